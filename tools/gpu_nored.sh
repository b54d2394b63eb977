mkdir -p gpurun_out
run() {
  for c in 0 112 128 144; do timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 4096 --ctas $c; done
  for c in 0 128 144; do timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 4096 --n 6144 --ctas $c; done
  for c in 0 128; do timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 32 --m 14336 --n 4096 --ctas $c; done
}
echo "== normal"; run
MESW_XFLAGS="-DMESW_EXP_NORED" python build.py --force > /dev/null 2>&1
echo "== NORED"; run
