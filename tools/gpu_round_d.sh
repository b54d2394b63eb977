mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d_pytest.log 2>&1; echo "rc $?" >> gpurun_out/d_pytest.log
bash tools/kb_quick.sh > gpurun_out/d_kb.log 2>&1
timeout 60 python tools/kbench.py --reps 50 --experts 16 --batch 32 >> gpurun_out/d_kb.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/d_c2.log 2>&1
timeout 300 python bench.py --experts 16 --batch 128 --steps 10 --no-cpu-baseline > gpurun_out/d_c3.log 2>&1
