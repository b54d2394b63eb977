mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/k_prefill.log 2>&1; echo "rc $?" >> gpurun_out/k_prefill.log
timeout 120 python tools/prefill_bench.py > gpurun_out/k_pfb.log 2>&1
timeout 120 python tools/prefill_bench.py 14336 4096 16 2048 >> gpurun_out/k_pfb.log 2>&1
timeout 120 python tools/prefill_bench.py 4096 14336 16 4096 >> gpurun_out/k_pfb.log 2>&1
