"""Kernel micro-benchmark for the fused multi-expert linear (CUDA-event timed).

    python tools/kbench.py [--m 4096 --n 14336 --experts 3 --batch 8 --reps 50]
Prints one line per configuration with us/launch and algorithmic GB/s.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2406_09041_b200 import compress, synth
from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, LinearPlan,
                                           align_segments, corr_table, pack_x)


def make(m, n, E, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    geom = LinearGeometry(m, (n,))
    dw = DeviceWeight.empty(geom)
    w = (torch.randn((m, n), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    dw.load_block(0, w)
    del w
    table = ExpertTable("cuda")
    for e in range(E):
        blob = synth.synthetic_expert_artifact(seed * 100 + e, [(m, n)], f"e{e}")
        table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(blob).layers[0]], geom))
    return geom, dw, table


def run(m, n, E, B, reps, base=True, replicas=3, num_ctas=0, offset=True):
    """Times the kernel alone: expert groups are laid out on 16-row boundaries (as the
    serving engine does) and each launch is a pre-built LinearPlan."""
    sets = [make(m, n, E, r) for r in range(replicas)]
    per = [B // E + (1 if i < B % E else 0) for i in range(E)] if E else []
    segs, cur = [], 0
    for e, c in enumerate(per):
        if c:
            segs.append((cur, cur + c, e))
        cur += c
    rows, asegs, _ = align_segments(B, segs)
    x = (torch.randn((rows, m), device="cuda")).to(torch.bfloat16)
    corr = corr_table(rows, m, "cuda") if offset else None
    xc = pack_x(x, corr=corr)
    y = torch.empty((rows, n), dtype=torch.bfloat16, device="cuda")
    plans = [LinearPlan(xc, rows, dw if base else None, table if E else None, asegs, y, geom=geom,
                        num_ctas=num_ctas, x_corr=corr) for geom, dw, table in sets]

    for i in range(5):
        plans[i % replicas]()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for i in range(reps):
        plans[i % replicas]()
    en.record()
    torch.cuda.synchronize()
    us = st.elapsed_time(en) * 1e3 / reps
    nbytes = synth.linear_bytes(m, n, E, B, base=base)
    print(f"m={m} n={n} E={E} B={B} rows={rows} base={base} ctas={num_ctas} off={int(offset)}: {us:8.2f} us  "
          f"{nbytes/us/1e3:8.1f} GB/s ({nbytes/us/1e3/6549.8*100:5.1f}% of 6549.8)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--n", type=int, default=14336)
    ap.add_argument("--experts", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--ab", action="store_true")
    a = ap.parse_args()
    if a.sweep:
        for (m, n) in [(4096, 14336), (4096, 6144), (4096, 4096), (14336, 4096), (4096, 28672)]:
            run(m, n, 0, 8, a.reps)
            run(m, n, 3, 8, a.reps)
        for B in (1, 16, 32, 64):
            run(4096, 14336, 3, B, a.reps)
        run(4096, 14336, 16, 32, a.reps)
        run(4096, 14336, 3, 8, a.reps, base=False)
    elif a.ab:  # exact vs offset-form code expansion on the headline shapes
        for (m, n, E, B) in [(4096, 14336, 3, 8), (4096, 6144, 3, 32), (14336, 4096, 3, 32), (4096, 28672, 3, 32),
                             (4096, 4096, 3, 32), (4096, 14336, 16, 64)]:
            run(m, n, E, B, a.reps, offset=False)
            run(m, n, E, B, a.reps, offset=True)
    else:
        run(a.m, a.n, a.experts, a.batch, a.reps, num_ctas=a.ctas, offset=not a.exact)
