mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_glue.py tests/test_gpu_corr.py tests/test_gpu_mistral.py tests/test_gpu_mistral_full.py -x -q -p no:cacheprovider > gpurun_out/attn_pytest.log 2>&1
timeout 120 python tools/attn_bench.py > gpurun_out/attn_b.log 2>&1
for s in "" attn; do timeout 300 python tools/skip_glue.py --skip "$s"; done > gpurun_out/attn_skip.log 2>&1
