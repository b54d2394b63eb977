# A/B: even A sub-rings (default) vs odd ones (MESW_ODD_SLOTS=1) on the C1/C2 linear shapes.
for ODD in "" 1; do
  echo "== MESW_ODD_SLOTS=$ODD"
  if [ -n "$ODD" ]; then export MESW_ODD_SLOTS=1; fi; bash tools/kb_quick.sh
done
