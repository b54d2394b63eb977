# Round-end measurement pass on one B200 (run under gpurun); outputs to gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/f_pytest.log
timeout 600 python bench.py > gpurun_out/f_c2.log 2>&1
timeout 300 python bench.py --config c1 > gpurun_out/f_c1.log 2>&1
timeout 600 python bench.py --experts 16 --batch 32 --no-cpu-baseline > gpurun_out/f_c3_32.log 2>&1
timeout 600 python bench.py --experts 16 --batch 128 --no-cpu-baseline > gpurun_out/f_c3_128.log 2>&1
timeout 300 python bench.py --config c4 > gpurun_out/f_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_c5.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1
# launch list of one decode step (C2, B=32, 3 experts), then one full capture of the C1 kernel
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/f_c2_launches.csv python tools/profile_step.py --batch 32 > gpurun_out/f_ncu_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:me_linear -s 2 -c 1 \
  -o gpurun_out/f_c1 -f python tools/one_launch.py 4096 14336 3 8 142 > gpurun_out/f_ncu_c1.log 2>&1
echo done
