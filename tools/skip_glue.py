"""Timing experiment: the C2 decode step (graph replay) with some glue launches removed.

    python tools/skip_glue.py [--skip norm,swiglu,attn]

The skipped kernels' outputs are stale, so the tokens are garbage: this only bounds what
fusing those launches into the fused linears could save."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench_mistral as bm
from paper_2406_09041_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--experts", type=int, default=3)
ap.add_argument("--skip", default="")
a = ap.parse_args()
L = _lib.lib()
names = {"norm": ["mesw_rmsnorm"], "swiglu": ["mesw_swiglu"],
         "attn": ["mesw_attention_decode_rope", "mesw_attention_decode"]}
E = a.experts
eng = bm.build_engine(a.batch, list(range(E)), [i % E for i in range(a.batch)], max_batch=a.batch + 16 * E)
eng.wrap_positions = True
for k in [s for s in a.skip.split(",") if s]:
    for fn in names[k]:
        setattr(L, fn, lambda *args: 0)
eng.capture()
for _ in range(5):
    eng.replay()
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(30):
    eng.replay()
en.record()
torch.cuda.synchronize()
ms = st.elapsed_time(en) / 30
print(f"skip={a.skip or '-':20s} {ms:7.3f} ms/step  {a.batch / ms * 1e3:8.1f} tok/s")
