mkdir -p gpurun_out
MESW_PROFILE=1 MESW_XFLAGS="-DMESW_EXP_WARM" python build.py --force > /dev/null 2>&1
cd tools; ALIGNED=1 timeout 120 python ktiming.py 4096 14336 3 8 > ../gpurun_out/warm_c1.log 2>&1
ALIGNED=1 timeout 120 python ktiming.py 4096 4096 3 32 > ../gpurun_out/warm_o.log 2>&1
