"""One fused-linear configuration launched a few times (for ncu / sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_09041_b200.device import LinearPlan, align_segments, corr_table, pack_x
from kbench import make
m, n, E, B = (int(v) for v in sys.argv[1:5])
ctas = int(sys.argv[5]) if len(sys.argv) > 5 else 0
geom, dw, table = make(m, n, max(E, 1), 0)
per = [B // E + (1 if i < B % E else 0) for i in range(E)] if E else []
segs, cur = [], 0
for e, c in enumerate(per):
    if c:
        segs.append((cur, cur + c, e))
    cur += c
rows, asegs, _ = align_segments(B, segs)
x = torch.randn((rows, m), device="cuda").to(torch.bfloat16)
y = torch.empty((rows, n), dtype=torch.bfloat16, device="cuda")
corr = corr_table(rows, m, "cuda")  # offset-form codes, as the serving engine runs them
plan = LinearPlan(pack_x(x, corr=corr), rows, dw, table if E else None, asegs, y, geom=geom, x_corr=corr,
                  num_ctas=ctas)
for _ in range(4):
    plan()
torch.cuda.synchronize()
print("ok", rows)
