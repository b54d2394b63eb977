mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_toy.py tests/test_gpu_glue.py tests/test_gpu_corr.py -q -x > gpurun_out/r_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/r_c1.log 2>&1
