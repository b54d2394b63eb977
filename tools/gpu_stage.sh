mkdir -p gpurun_out
for v in 0 4 8; do
  MESW_XFLAGS="-DMESW_STAGE_MIN=$v" python build.py --force > /dev/null 2>&1
  echo "== MESW_STAGE_MIN=$v"; bash tools/kb_quick.sh
done > gpurun_out/stage_kb.log 2>&1
