mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_mistral.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1
(bash tools/kb_quick.sh; timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 4096 --ctas 128; timeout 60 python tools/kbench.py --reps 30 --experts 16 --batch 128 --m 4096 --n 28672) > gpurun_out/q_kb.log 2>&1
