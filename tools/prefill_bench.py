"""K3 prefill kernel timing: T tokens over E experts (128-token groups) through one linear
(CUDA events, L2-cold rotation over 2 weight/expert replicas), and the base-only form.

    python tools/prefill_bench.py [m n E T]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from paper_2406_09041_b200.device import PrefillPlan, pack_x  # noqa: E402
from kbench import make  # noqa: E402

m, n, E, T = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 14336, 16, 2048)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["bf16_tflops"]
sets = [make(m, n, E, r) for r in range(2)]
x = torch.randn((T, m), device="cuda").to(torch.bfloat16)
xc = pack_x(x)
y = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
groups = T // 128
for label, slots in (("fused", [g * E // groups for g in range(groups)]), ("base-only", [-1] * groups)):
    plans = [PrefillPlan(xc, T, T, dw, table, slots, y) for geom, dw, table in sets]
    for i in range(4):
        plans[i % 2]()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    st.record()
    for i in range(reps):
        plans[i % 2]()
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / reps
    tf = 2.0 * T * m * n / (ms / 1e3) / 1e12
    print(f"{label:9s} m={m} n={n} E={E} T={T}: {ms * 1e3:8.1f} us  {tf:7.1f} TFLOP/s base-equivalent "
          f"({tf / peak:.3f} of {peak} burst)", flush=True)
