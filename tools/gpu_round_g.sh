mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_corr.py tests/test_gpu_toy.py -q -x > gpurun_out/g_pytest.log 2>&1; echo "rc $?" >> gpurun_out/g_pytest.log
bash tools/kb_quick.sh > gpurun_out/g_kb.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-extras > gpurun_out/g_c2.log 2>&1
for B in 1 2 4; do MESW_XFLAGS="-DMESW_DQ_BATCH=$B" python build.py --force > /dev/null 2>&1; echo "== batch $B" >> gpurun_out/g_kbb.log; timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 8 >> gpurun_out/g_kbb.log 2>&1; timeout 60 python tools/kbench.py --reps 100 --experts 8 --batch 16 >> gpurun_out/g_kbb.log 2>&1; NOBASE=1 timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 28672 >> gpurun_out/g_kbb.log 2>&1; done
