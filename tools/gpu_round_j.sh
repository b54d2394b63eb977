mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/j_prefill.log 2>&1; echo "rc $?" >> gpurun_out/j_prefill.log
timeout 120 python tools/prefill_bench.py > gpurun_out/j_pfb.log 2>&1
timeout 120 python tools/prefill_bench.py 4096 4096 16 2048 >> gpurun_out/j_pfb.log 2>&1
timeout 120 python tools/prefill_bench.py 14336 4096 16 2048 >> gpurun_out/j_pfb.log 2>&1
timeout 300 python bench.py --config c4 --steps 10 > gpurun_out/j_c4.log 2>&1
