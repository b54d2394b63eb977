mkdir -p gpurun_out
for s in "" norm swiglu attn "norm,swiglu" "norm,swiglu,attn"; do timeout 300 python tools/skip_glue.py --skip "$s"; done > gpurun_out/skip_glue.log 2>&1
