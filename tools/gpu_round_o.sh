mkdir -p gpurun_out
cd tools
timeout 120 python prefill_bench.py > ../gpurun_out/o_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill -s 3 -c 1 \
  -o ../gpurun_out/o_pf -f python prefill_bench.py > ../gpurun_out/o_ncu.log 2>&1
