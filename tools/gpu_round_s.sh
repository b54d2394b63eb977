mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_toy.py tests/test_gpu_corr.py tests/test_gpu_mistral.py -q -x > gpurun_out/s_pytest.log 2>&1; echo "rc $?" >> gpurun_out/s_pytest.log
bash tools/kb_quick.sh > gpurun_out/s_kb.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/s_c1.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-extras > gpurun_out/s_c2.log 2>&1
