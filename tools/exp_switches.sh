# Experiment driver: rebuild with MESW_XFLAGS switches and time C1-like shapes (tools/kbench.py).
for X in "" "-DMESW_EXP_NODQ -DMESW_EXP_NOMMA"; do
  MESW_XFLAGS="$X" python build.py --force > /dev/null 2>&1 || echo BUILD FAIL
  echo "== $X"
  for n in 7168 14336 28672 57344; do
    timeout 60 python tools/kbench.py --reps 100 --m 4096 --n $n --batch 8
    timeout 60 python tools/kbench.py --reps 100 --m 4096 --n $n --batch 8 --experts 0
  done
done
