# Launch-group sizing for many-expert batches: per-expert cost vs windows per launch and
# accumulator double-buffering (MESW_NACC=1 trades it for A-ring slots).
for EB in "4 8" "6 12" "8 16" "12 24"; do
  set -- $EB
  timeout 60 python tools/kbench.py --reps 100 --experts $1 --batch $2
  MESW_NACC=1 timeout 60 python tools/kbench.py --reps 100 --experts $1 --batch $2
done
