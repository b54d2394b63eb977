# half-jobs build: correctness + kernel timings; then profile builds (cycle counters)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_corr.py tests/test_gpu_toy.py -q -x > gpurun_out/f_pytest.log 2>&1; echo "rc $?" >> gpurun_out/f_pytest.log
bash tools/kb_quick.sh > gpurun_out/f_kb.log 2>&1
MESW_PROFILE=1 python build.py --force > gpurun_out/f_build.log 2>&1
cd tools
timeout 120 python ktiming.py 4096 14336 12 178 > ../gpurun_out/f_kt12.log 2>&1
timeout 120 python ktiming.py 4096 14336 3 34 > ../gpurun_out/f_kt3.log 2>&1
NOBASE=1 timeout 120 python ktiming.py 4096 14336 3 34 > ../gpurun_out/f_kt3nb.log 2>&1
