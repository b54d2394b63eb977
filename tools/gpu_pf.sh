mkdir -p gpurun_out
for cfg in "2 4" "3 3"; do
  set -- $cfg
  MESW_XFLAGS="-DMESW_PF_NW=$1 -DMESW_PF_NX=$2" python build.py --force > /dev/null 2>&1
  echo "== NW=$1 NX=$2"
  (cd tools && timeout 120 python prefill_bench.py && timeout 120 python pf_timing.py)
done > gpurun_out/pf_ab.log 2>&1
