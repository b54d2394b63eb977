# profile pass: STTM micro + per-role cycle counters of many-expert K2 launches
mkdir -p gpurun_out
./tools/micro/sttm_rate > gpurun_out/b_sttm.log 2>&1
MESW_PROFILE=1 python build.py --force > gpurun_out/b_build.log 2>&1
cd tools
timeout 120 python ktiming.py 4096 14336 12 178 > ../gpurun_out/b_kt12.log 2>&1
timeout 120 python ktiming.py 4096 14336 4 52 > ../gpurun_out/b_kt4.log 2>&1
timeout 120 python ktiming.py 4096 14336 3 34 > ../gpurun_out/b_kt3.log 2>&1
