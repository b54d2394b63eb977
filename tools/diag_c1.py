import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_09041_b200.device import LinearPlan, pack_x
from kbench import make
m, n = int(sys.argv[1]), int(sys.argv[2])
geom, dw, table = make(m, n, 3, 0)
W = dw.dense().double()
R = [table.deltas[e].reconstruct().double() for e in range(3)]
for label, segs, rows, ctas in [("E0 r34", [], 34, 0), ("E1 r8", [(0, 8, 0)], 8, 0), ("E1 r34", [(0, 34, 0)], 34, 0),
                                ("E3 r34", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34, 0),
                                ("E3 r34 G=1", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34, 1),
                                ("E3 r34 G=7", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34, 7)]:
    x = torch.randn((rows, m), device="cuda").to(torch.bfloat16)
    y = torch.empty((rows, n), dtype=torch.float32, device="cuda")
    LinearPlan(pack_x(x), rows, dw, table if segs else None, segs, y, geom=geom, num_ctas=ctas)()
    torch.cuda.synchronize()
    ref = x.double() @ W
    for b, e, sl in segs:
        ref[b:e] += x[b:e].double() @ R[sl]
    err = (y.double() - ref).abs()
    rel = (err.max() / ref.abs().max()).item()
    rows_bad = (err.max(1).values > 1e-3 * ref.abs().max()).nonzero().flatten().tolist()
    cols_bad = (err.max(0).values > 1e-3 * ref.abs().max()).nonzero().flatten()
    print(f"{label:12s} rel {rel:.2e} bad rows {rows_bad[:12]} n_bad_cols {cols_bad.numel()} first {cols_bad[:8].tolist()}", flush=True)
