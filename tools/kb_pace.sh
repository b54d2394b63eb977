# A/B: base-issuer pacing (MESW_DBG = lag + 1) on the headline and many-expert shapes.
for D in 0 1 2 3; do
  echo "== MESW_DBG=$D"
  MESW_DBG=$D bash tools/kb_quick.sh
done
