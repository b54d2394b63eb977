# ncu source-level capture of a 12-expert K2 launch (where do the dequant warps stall?)
mkdir -p gpurun_out
cd tools
timeout 120 python one_launch.py 4096 14336 12 24 > ../gpurun_out/c_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:me_linear -s 2 -c 1 \
  -o ../gpurun_out/c_e12 -f python one_launch.py 4096 14336 12 24 > ../gpurun_out/c_ncu.log 2>&1
