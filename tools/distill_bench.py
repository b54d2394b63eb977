"""f3 measurement: the per-layer quantizer kernels of step-size distillation on one
Mistral-shaped layer (default 4096 x 14336, b=2, k=8), against the reference algorithm
(oracle/distill.py, numpy) on the host for the same layer.

  mesw_ste_reconstruct  W_eff = W + reconstruct(steps)   bytes: delta + W read, W_eff write (12 B/elem)
  mesw_ste_step_grad    grad = STE contraction            bytes: delta + upstream read (8 B/elem)

Prints one JSON line.  Times are CUDA events over `reps` launches after warm-up.
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_09041_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--n", type=int, default=14336)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cpu", action="store_true", help="also time the numpy reference algorithm")
    a = ap.parse_args()
    m, n, k, bits = a.m, a.n, 8, 2
    L = _lib.lib()
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    delta = torch.randn((m, n), generator=g, device="cuda") * 1e-3
    w = torch.randn((m, n), generator=g, device="cuda") * 0.02
    up = torch.randn((m, n), generator=g, device="cuda")
    steps = (delta.abs().amax(dim=0) / 1.0).contiguous()
    slot = torch.full((m,), -1, dtype=torch.int32, device="cuda")
    idx = torch.arange(0, m, m // k, device="cuda")[:k]
    slot[idx] = torch.arange(k, dtype=torch.int32, device="cuda")
    rows = (torch.randn((k, n), generator=g, device="cuda") * 0.05).half().float()
    out = torch.empty_like(w)
    grad = torch.empty(n, dtype=torch.float32, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def rec():
        _lib.check(L.mesw_ste_reconstruct(delta.data_ptr(), m, n, steps.data_ptr(), bits, slot.data_ptr(),
                                          rows.data_ptr(), w.data_ptr(), out.data_ptr(), s))

    def grd():
        _lib.check(L.mesw_ste_step_grad(delta.data_ptr(), m, n, steps.data_ptr(), bits, slot.data_ptr(),
                                        up.data_ptr(), grad.data_ptr(), s))

    res = {"workload": f"f3 one layer {m}x{n} b={bits} k={k}"}
    peak = 6549.8
    for name, fn, bpe in (("ste_reconstruct", rec, 12), ("ste_step_grad", grd, 8)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        gbs = bpe * m * n / us / 1e3
        res[name] = {"us": round(us, 2), "GB/s": round(gbs, 1), "frac_hbm": round(gbs / peak, 3)}
    if a.cpu:
        from oracle import distill as od  # the checker/baseline only
        d_np, up_np, st_np = delta.cpu().numpy(), up.cpu().numpy(), steps.cpu().numpy()
        st = od.LayerState(d_np, idx.cpu().numpy(), rows.cpu().numpy(), st_np, bits)
        t0 = time.perf_counter()
        st.reconstruct()
        t1 = time.perf_counter()
        g_ref = st.step_gradient(up_np)
        t2 = time.perf_counter()
        res["cpu_reference"] = {"reconstruct_s": round(t1 - t0, 3), "step_grad_s": round(t2 - t1, 3),
                                "threads": os.cpu_count(), "kind": "port (numpy)"}
        res["step_grad_bit_exact"] = bool(np.array_equal(grad.cpu().numpy(), g_ref))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
