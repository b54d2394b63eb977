# Experiment driver (many-expert launches): rebuild with MESW_XFLAGS switches and time
# 12- and 8-expert windows per launch (tools/kbench.py).
for X in "" "-DMESW_EXP_NODQ" "-DMESW_EXP_NOMMA" "-DMESW_EXP_NODQ -DMESW_EXP_NOMMA" "-DMESW_EXP_ST1"; do
  MESW_XFLAGS="$X" python build.py --force > /dev/null 2>&1 || echo BUILD FAIL
  echo "== $X"
  timeout 60 python tools/kbench.py --reps 100 --experts 12 --batch 24
  timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 8
done
for S in 1 2 3; do
  echo "== MESW_MAXSLOTS=$S"
  MESW_MAXSLOTS=$S timeout 60 python tools/kbench.py --reps 100 --experts 3 --batch 8
  MESW_MAXSLOTS=$S timeout 60 python tools/kbench.py --reps 100 --experts 4 --batch 8
done
python build.py --force > /dev/null 2>&1
