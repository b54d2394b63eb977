# A/B timing of the fused linear on the C3 (16 experts, B=128) and C2 (3 experts, B=32) shapes.
for s in "4096 6144" "4096 4096" "4096 28672" "14336 4096"; do
  set -- $s
  timeout 60 python tools/kbench.py --reps 50 --experts 16 --batch 128 --m $1 --n $2
  timeout 60 python tools/kbench.py --reps 50 --experts 16 --batch 32 --m $1 --n $2
  timeout 60 python tools/kbench.py --reps 50 --experts 3 --batch 32 --m $1 --n $2
done
