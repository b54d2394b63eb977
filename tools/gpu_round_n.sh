mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/n_prefill.log 2>&1; echo "rc $?" >> gpurun_out/n_prefill.log
timeout 120 python tools/prefill_bench.py > gpurun_out/n_pfb.log 2>&1
timeout 120 python tools/prefill_bench.py 14336 4096 16 2048 >> gpurun_out/n_pfb.log 2>&1
cd tools; timeout 120 python pf_timing.py > ../gpurun_out/n_pft.log 2>&1
