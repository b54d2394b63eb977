# Quick A/B timing of the fused linear on the headline and many-expert shapes.
timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 8
timeout 60 python tools/kbench.py --reps 100 --experts 12 --batch 24
timeout 60 python tools/kbench.py --reps 100 --experts 8 --batch 16
timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 28672
timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 14336 --n 4096
timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 6144
timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 4096
