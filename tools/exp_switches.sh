# Experiment driver: rebuild with MESW_XFLAGS switches and time C1-like shapes (tools/kbench.py).
for X in "" "-DMESW_EXP_ST1" "-DMESW_EXP_KH=1" "-DMESW_EXP_NODQ"; do
  MESW_XFLAGS="$X" python build.py --force > /dev/null 2>&1 || echo BUILD FAIL
  echo "== $X"
  timeout 60 python tools/kbench.py --reps 200
  timeout 60 python tools/kbench.py --reps 200 --m 4096 --n 28672 --batch 32
done
python build.py --force > /dev/null 2>&1
