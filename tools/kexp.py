"""Ad-hoc kernel experiments (timing only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_09041_b200 import synth
from paper_2406_09041_b200.device import LinearPlan, pack_x
from kbench import make

def t(plans, reps=20):
    for i in range(5): plans[i % len(plans)]()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for i in range(reps): plans[i % len(plans)]()
    en.record(); torch.cuda.synchronize()
    return st.elapsed_time(en) * 1e3 / reps

m, n = 4096, 14336
sets = [make(m, n, 3, r) for r in range(3)]
def run(label, segs, rows, base=True, same=False):
    x = torch.randn((rows, m), device="cuda").to(torch.bfloat16)
    xc = pack_x(x)
    y = torch.empty((rows, n), dtype=torch.bfloat16, device="cuda")
    ss = [(b, e, 0 if same else sl) for b, e, sl in segs]
    plans = [LinearPlan(xc, rows, dw if base else None, table if segs else None, ss, y, geom=geom) for geom, dw, table in sets]
    print(f"{label:40s} {t(plans):8.2f} us", flush=True)

run("E0 rows8", [], 8)
run("E0 rows48", [], 48)
run("E1 rows8", [(0, 8, 0)], 8)
run("E1 rows48", [(0, 48, 0)], 48)
run("E3 rows34 distinct", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34)
run("E3 rows34 same-expert", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34, same=True)
run("E3 rows34 delta-only", [(0, 3, 0), (16, 19, 1), (32, 34, 2)], 34, base=False)
run("E2 rows18", [(0, 3, 0), (16, 18, 1)], 18)
