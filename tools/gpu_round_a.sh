mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_corr.py -q -x > gpurun_out/a_pytest.log 2>&1; echo "rc $?" >> gpurun_out/a_pytest.log
bash tools/kb_quick.sh > gpurun_out/a_kb.log 2>&1
timeout 60 python tools/kbench.py --reps 50 --experts 16 --batch 32 >> gpurun_out/a_kb.log 2>&1
timeout 60 python tools/kbench.py --reps 50 --experts 12 --batch 96 >> gpurun_out/a_kb.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/a_c2.log 2>&1
timeout 300 python bench.py --experts 16 --batch 128 --steps 10 --no-cpu-baseline > gpurun_out/a_c3.log 2>&1
