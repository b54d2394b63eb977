"""Issuer-side cycle breakdown of one K3 prefill launch (MESW_PF_PROF=1)."""
import ctypes as C
import os
import sys
os.environ["MESW_PF_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2406_09041_b200 import _lib  # noqa: E402
from paper_2406_09041_b200.device import PrefillPlan, pack_x  # noqa: E402
from kbench import make  # noqa: E402

m, n, E, T = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 14336, 16, 2048)
base_only = len(sys.argv) > 5
geom, dw, table = make(m, n, E, 0)
x = torch.randn((T, m), device="cuda").to(torch.bfloat16)
y = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
groups = T // 128
slots = [-1] * groups if base_only else [g * E // groups for g in range(groups)]
plan = PrefillPlan(pack_x(x), T, T, dw, table, slots, y)
for _ in range(3):
    plan()
torch.cuda.synchronize()
L = _lib.lib()
L.mesw_prefill_profile_copy.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(1024 * 8, np.uint64)
_lib.check(L.mesw_prefill_profile_copy(buf.ctypes.data, 1024))
pr = buf.reshape(1024, 8)[:74, :5].astype(np.int64)
names = ["wait_accempty", "wait_x", "wait_A", "issue", "total"]
print(f"m={m} n={n} E={E} T={T} base_only={base_only}: per leader issuer (SM cycles), median / max over pairs")
for i, nm in enumerate(names):
    print(f"  {nm:14s} {np.median(pr[:, i]):12.0f} {pr[:, i].max():12.0f}")
