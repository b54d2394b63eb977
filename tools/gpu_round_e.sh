mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router.py tests/test_gpu_mistral.py tests/test_gpu_mistral_full.py -q -x -s > gpurun_out/e_pytest.log 2>&1; echo "rc $?" >> gpurun_out/e_pytest.log
timeout 900 python bench.py > gpurun_out/e_bench.log 2> gpurun_out/e_bench.err; echo "rc $?" >> gpurun_out/e_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/e_ref.log 2> gpurun_out/e_ref.err; echo "rc $?" >> gpurun_out/e_ref.err
