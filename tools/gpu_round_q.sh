mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "rc $?" >> gpurun_out/q_pytest.log
