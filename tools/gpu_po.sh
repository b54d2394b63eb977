mkdir -p gpurun_out
MESW_PROFILE=1 python build.py --force > /dev/null 2>&1
cd tools; CTAS=128 ALIGNED=1 timeout 120 python ktiming.py 4096 4096 3 32 > ../gpurun_out/po_o.log 2>&1
