# Round-end measurement pass on one B200 (run under gpurun); outputs to gpurun_out/final_*.
# Plain runs first; the ncu passes re-run the same command lines after they exited 0.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 600 python bench.py --config c4 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 600 python bench.py --config c1 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
# launch lists with per-launch DRAM bytes: one C2 decode step (B=32, 3 experts), one C3 step (B=128, 16 experts)
timeout 600 python tools/profile_step.py --batch 32 --experts 3 > gpurun_out/final_ps_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/final_c2_launches.csv python tools/profile_step.py --batch 32 --experts 3 \
  > gpurun_out/final_ncu_c2.log 2>&1
timeout 900 python tools/profile_step.py --batch 128 --experts 16 > gpurun_out/final_ps_c3.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/final_c3_launches.csv python tools/profile_step.py --batch 128 --experts 16 \
  > gpurun_out/final_ncu_c3.log 2>&1
# full captures of the dominant kernels: the C1 fused linear, the C4 prefill linear
cd tools
timeout 120 python one_launch.py 4096 14336 3 8 > ../gpurun_out/final_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:me_linear -s 2 -c 1 \
  -o ../gpurun_out/final_c1 -f python one_launch.py 4096 14336 3 8 > ../gpurun_out/final_ncu_c1.log 2>&1
timeout 120 python prefill_bench.py > ../gpurun_out/final_pfb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill -s 3 -c 1 \
  -o ../gpurun_out/final_pf -f python prefill_bench.py > ../gpurun_out/final_ncu_pf.log 2>&1
echo done
