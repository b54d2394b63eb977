# Round-end measurement pass on one B200 (run under gpurun); outputs to gpurun_out/${P}_*.
# Plain runs first; the ncu passes re-run the same command lines after they exited 0.
set -x
P=${P:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${P}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${P}_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/${P}_c2.json 2> gpurun_out/${P}_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/${P}_ref.json 2> gpurun_out/${P}_ref.err
timeout 600 python bench.py --config c4 > gpurun_out/${P}_c4.json 2> gpurun_out/${P}_c4.err
timeout 600 python bench.py --config c1 > gpurun_out/${P}_c1.json 2> gpurun_out/${P}_c1.err
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
# launch lists with per-launch DRAM bytes: one C2 decode step (B=32, 3 experts), one C3 step (B=128, 16 experts)
timeout 600 python tools/profile_step.py --batch 32 --experts 3 > gpurun_out/${P}_ps_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${P}_c2_launches.csv python tools/profile_step.py --batch 32 --experts 3 \
  > gpurun_out/${P}_ncu_c2.log 2>&1
timeout 900 python tools/profile_step.py --batch 128 --experts 16 > gpurun_out/${P}_ps_c3.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${P}_c3_launches.csv python tools/profile_step.py --batch 128 --experts 16 \
  > gpurun_out/${P}_ncu_c3.log 2>&1
# full captures of the dominant kernels: the C1 fused linear, the C4 prefill linear
cd tools
timeout 120 python one_launch.py 4096 14336 3 8 > ../gpurun_out/${P}_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:me_linear -s 2 -c 1 \
  -o ../gpurun_out/${P}_c1 -f python one_launch.py 4096 14336 3 8 > ../gpurun_out/${P}_ncu_c1.log 2>&1
timeout 120 python prefill_bench.py > ../gpurun_out/${P}_pfb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill -s 3 -c 1 \
  -o ../gpurun_out/${P}_pf -f python prefill_bench.py > ../gpurun_out/${P}_ncu_pf.log 2>&1
echo done
