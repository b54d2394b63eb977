mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x -s > gpurun_out/h_prefill.log 2>&1; echo "rc $?" >> gpurun_out/h_prefill.log
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_corr.py tests/test_gpu_toy.py -q -x > gpurun_out/h_pytest.log 2>&1; echo "rc $?" >> gpurun_out/h_pytest.log
bash tools/kb_quick.sh > gpurun_out/h_kb.log 2>&1
timeout 120 python tools/prefill_bench.py > gpurun_out/h_pfb.log 2>&1
