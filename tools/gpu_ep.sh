mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_mistral.py -x -q -p no:cacheprovider > gpurun_out/ep_pytest.log 2>&1
bash tools/kb_quick.sh > gpurun_out/ep_kb.log 2>&1
MESW_PROFILE=1 python build.py --force > /dev/null 2>&1
cd tools; ALIGNED=1 timeout 120 python ktiming.py 4096 14336 3 8 > ../gpurun_out/ep_c1.log 2>&1
