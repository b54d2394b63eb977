mkdir -p gpurun_out
for v in 0 1024; do
  MESW_XFLAGS="-DMESW_ATTN_SINGLE_MAX=$v" python build.py --force > /dev/null 2>&1
  echo "== SINGLE_MAX=$v"; timeout 120 python tools/attn_bench.py
done > gpurun_out/attn_ab.log 2>&1
