"""C4 probe: a 2048-token prefill through one fused linear (16 experts x 128 tokens)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_09041_b200.device import LinearPlan, MAX_ROWS, align_segments, pack_x, me_linear
from kbench import make

m, n, E, T = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 14336, 16, 2048)
geom, dw, table = make(m, n, E, 0)
per = T // E
x = torch.randn((T, m), device="cuda").to(torch.bfloat16)
y = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
# launch groups of <= MAX_ROWS rows, each a pre-built plan (expert groups already 16-aligned)
plans = []
for g0 in range(0, T, MAX_ROWS // per * per):
    g1 = min(T, g0 + MAX_ROWS // per * per)
    segs = [(s - g0, min(s + per, g1) - g0, (s // per)) for s in range(g0, g1, per)]
    xc = pack_x(x[g0:g1].contiguous())
    plans.append(LinearPlan(xc, g1 - g0, dw, table, segs, y[g0:g1], geom=geom))
for _ in range(3):
    for p in plans:
        p()
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(5):
    for p in plans:
        p()
en.record()
torch.cuda.synchronize()
ms = st.elapsed_time(en) / 5
flops = 2.0 * T * m * n * 2  # base + delta contraction
print(f"prefill T={T} E={E} {m}x{n}: {len(plans)} launches, {ms:.3f} ms, {flops / ms / 1e9:.1f} TFLOP/s "
      f"(base+delta), {flops / 2 / ms / 1e9:.1f} TFLOP/s base-only equivalent")
