"""Workload implementations for bench.py (kept separate so bench.py stays a thin contract shell).

`run_ours` times OUR GPU path; `reference_arm` times the reference's CPU algorithm
(the oracle port -- the reference is Python and cannot travel to the GPU box).
Only the cpu_baseline / reference legs import `oracle/`.
"""

from __future__ import annotations

import os
import time

import numpy as np

C1_M, C1_N, C1_E, C1_B, C1_K = 4096, 14336, 3, 8, 8


def _c1_segments(B: int, E: int):
    """Experts t mod E, grouped: returns (segments, order)."""
    expert_of = np.arange(B) % E
    order = np.argsort(expert_of, kind="stable")
    segs, cur = [], 0
    for e in range(E):
        c = int((expert_of == e).sum())
        if c:
            segs.append((cur, cur + c, e))
        cur += c
    return segs, order


def _c1_inputs(seed_base: int = 0):
    """Synthetic C1 weights / artifacts on the host (f32 W rounded to bf16 on upload)."""
    from paper_2406_09041_b200 import compress, synth
    rng = np.random.default_rng(seed_base)
    W = rng.normal(0, 0.02, size=(C1_M, C1_N)).astype(np.float32)
    arts = []
    for e in range(C1_E):
        blob = synth.synthetic_expert_artifact(1 + e + 100 * seed_base, [(C1_M, C1_N)], f"e{e}")
        arts.append(compress.deserialize_artifact(blob))
    x = np.random.default_rng(7).normal(0, 1, size=(C1_B, C1_M)).astype(np.float32)
    return W, arts, x


# ------------------------------------------------------------------ CPU (oracle) timing

def _cpu_c1_step(W, layers, x, segs, order):
    """Reference path as shipped: x@W + per expert group x_g @ reconstruct()."""
    y = x @ W
    xs = x[order]
    for (b, e, slot) in segs:
        y_g = xs[b:e] @ layers[slot].reconstruct()
        y[order[b:e]] += y_g
    return y


def _oracle_layers(arts):
    from oracle import mesw as om
    from paper_2406_09041_b200 import compress
    out = []
    for a in arts:
        _, ls = om.parse_artifact(compress.serialize_artifact(a))
        out.append(ls[0])
    return out


def cpu_c1_baseline(max_seconds: float = 20.0):
    W, arts, x = _c1_inputs()
    W = W.astype(np.float32)
    layers = _oracle_layers(arts)
    segs, order = _c1_segments(C1_B, C1_E)
    t0 = time.perf_counter()
    n = 0
    while True:
        _cpu_c1_step(W, layers, x, segs, order)
        n += 1
        if time.perf_counter() - t0 > max_seconds / 2 or n >= 3:
            break
    dt = (time.perf_counter() - t0) / n
    return dt, n


def reference_arm(args):
    import json  # noqa: F401
    cores = os.cpu_count()
    if args.config == "c1":
        W, arts, x = _c1_inputs()
        layers = _oracle_layers(arts)
        segs, order = _c1_segments(C1_B, C1_E)
        for _ in range(args.warmup):
            _cpu_c1_step(W, layers, x, segs, order)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _cpu_c1_step(W, layers, x, segs, order)
        dt = (time.perf_counter() - t0) / args.steps
        val = C1_B / dt
        return {"impl": "reference", "metric": "decode tokens/sec (one 4096x14336 linear, 3 mixed experts)",
                "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
                "config": {"workload": "c1: 4096x14336 linear, 3 experts b=2 k=8, batch 8 mixed decode"},
                "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port",
                                 "sample": "full C1 step: x@W + x_g@reconstruct() per expert group (numpy)"},
                "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if args.config == "c4":
        for _ in range(min(args.warmup, 1)):
            _c4_cpu()
        dts = [_c4_cpu() for _ in range(args.steps)]
        val = C4_T / (sum(dts) / len(dts))
        return {"impl": "reference", "metric": "prefill tokens/sec, one Mistral MLP linear 4096x14336, 2048 tokens over 16 experts",
                "value": val, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * C4_T / val, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": "c4: prefill 2048 tokens x 16 experts (128 each), 4096x14336 fused linear"},
                "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port",
                                 "sample": "per step: 1 expert group of 128 tokens (x_g@W + x_g@reconstruct), x16"},
                "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    from bench_mistral import reference_arm_c2
    return reference_arm_c2(args)


# ------------------------------------------------------------------ GPU timing

def _traffic(key):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/traffic.json), or None."""
    import json
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f)[key]["traffic"]
    except Exception:
        return None


def _device_c1(torch, W, arts, replicas: int):
    from paper_2406_09041_b200.device import DeviceDelta, DeviceWeight, ExpertTable
    sets = []
    for r in range(replicas):
        dw = DeviceWeight.from_dense([W])
        table = ExpertTable("cuda")
        for e, a in enumerate(arts):
            table.set(e, DeviceDelta.from_blocks([a.layers[0]]))
        sets.append((dw, table))
    return sets


def c1_leg(args, peaks):
    """BASELINE config 1 as an extra key of the default line (same process): kernel time,
    GB/s and roofline fraction of the fused linear, plus its delta-only (delta-GEMM) launch."""
    import argparse
    a = argparse.Namespace(**vars(args))
    a.no_cpu_baseline = True
    line = run_c1(a, 1, 0, 0, _NoClocks, peaks)
    return {"workload": line["config"]["workload"], "us_per_launch": line["ms_per_step"] * 1e3,
            "value": line["value"], "unit": "tokens/s", "roofline": line["roofline"],
            "delta_gemm": line["delta_gemm"], "e2e": line["e2e"], "num_ctas": line["config"]["num_ctas"]}


class _NoClocks:
    def __init__(self, *a):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampled by the main line"]}


def run_c1(args, ws, rank, local, ClockSampler, peaks):
    import torch
    from paper_2406_09041_b200 import synth
    from paper_2406_09041_b200.device import me_linear
    W, arts, x_np = _c1_inputs(seed_base=rank)
    replicas = 3  # rotate weight copies: 3 x 163 MB > 126 MB L2, no cross-step L2 reuse
    sets = _device_c1(torch, W, arts, replicas)
    segs, order = _c1_segments(C1_B, C1_E)
    x = torch.from_numpy(x_np[order]).to(torch.bfloat16).cuda()
    y = torch.empty((C1_B, C1_N), dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()
    # device-resident timing: the serving engine's form -- expert groups on 16-row boundaries,
    # activations already in the canonical tile layout, one pre-built launch per replica
    from paper_2406_09041_b200.device import LinearPlan, align_segments, corr_table, pack_x
    rows, asegs, src = align_segments(C1_B, segs)
    xa = torch.zeros((rows, C1_M), dtype=torch.bfloat16, device="cuda")
    src_t = torch.as_tensor(src, dtype=torch.int64, device="cuda")
    xa[src_t >= 0] = x[src_t[src_t >= 0]]
    corr = corr_table(rows, C1_M, "cuda")  # offset-code bias table, written with the canonical x
    xc = pack_x(xa, corr=corr)
    ya = torch.empty((rows, C1_N), dtype=torch.bfloat16, device="cuda")
    from paper_2406_09041_b200.device import Workspace, cta_candidates, tune_num_ctas
    dw0, tab0 = sets[0]
    scratch = torch.empty_like(ya)
    ctas = tune_num_ctas(("c1", rows, tuple(asegs)), lambda c: LinearPlan(xc, rows, dw0, tab0, asegs, scratch,
                                                                       x_corr=corr, num_ctas=c),
                         cta_candidates(dw0.geom, Workspace.get("cuda").sms))
    plans = [LinearPlan(xc, rows, dw, table, asegs, ya, x_corr=corr, num_ctas=ctas) for dw, table in sets]

    def step(i):
        plans[i % replicas]()

    # the timed region replays one CUDA graph holding all K launches (no host launch gaps)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        graph.capture_begin()
        for i in range(args.steps):
            plans[i % replicas](cs)
        graph.capture_end()
    torch.cuda.current_stream().wait_stream(cs)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph.replay()  # one untimed replay
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        st.record(stream)
        graph.replay()
        en.record(stream)
        torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    ms_t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    per_step = ms / args.steps
    tok_s = ws * C1_B * args.steps / (ms / 1e3)
    bytes_launch = synth.linear_bytes(C1_M, C1_N, C1_E, C1_B)
    peak, peak_kind = peaks()
    achieved = bytes_launch / (per_step / 1e3) / 1e9

    # delta-GEMM: the same launches without the base weight (codes + salient + steps only)
    dplans = [LinearPlan(xc, rows, None, table, asegs, ya, x_corr=corr, num_ctas=ctas) for _, table in sets]
    for i in range(args.warmup):
        dplans[i % replicas]()
    torch.cuda.synchronize()
    st.record(stream)
    for i in range(args.steps):
        dplans[i % replicas]()
    en.record(stream)
    torch.cuda.synchronize()
    d_us = st.elapsed_time(en) * 1e3 / args.steps
    d_bytes = synth.linear_bytes(C1_M, C1_N, C1_E, C1_B, base=False)
    d_gbs = d_bytes / (d_us / 1e6) / 1e9

    # e2e through the public API: pinned host x -> device, fused linear, y -> pinned host
    xh = torch.from_numpy(x_np[order]).to(torch.bfloat16).pin_memory()
    yh = torch.empty((C1_B, C1_N), dtype=torch.bfloat16).pin_memory()
    xd = torch.empty_like(x)
    for i in range(args.warmup):
        xd.copy_(xh, non_blocking=True)
        dw, table = sets[i % replicas]
        me_linear(xd, dw, table, segs, out=y, offset_codes=True)
        yh.copy_(y, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        xd.copy_(xh, non_blocking=True)
        dw, table = sets[i % replicas]
        me_linear(xd, dw, table, segs, out=y, offset_codes=True)
        yh.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    line = {
        "metric": "decode tokens/sec, one Mistral MLP linear 4096x14336 with 3 mixed experts; delta-GEMM HBM GB/s",
        "value": tok_s, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c1: 4096x14336 linear, 3 experts (b=2, k=8 fp16 salient), batch 8 mixed decode",
                   "l2": "3 rotating weight/delta replicas (489 MB) > 126 MB L2",
                   "parallelism": f"expert-sharded replicas x{ws}"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic("c1"), "peak_kind": peak_kind,
                     "bytes_per_launch": bytes_launch, "kernel": "me_linear_tc_kernel<2, true> (cta_group::2 pairs, offset-form codes)"},
        "e2e": {"value": ws * C1_B / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(xh.numel() * 2),
                "d2h_bytes_per_step": int(yh.numel() * 2)},
        "delta_gemm": {"bytes_per_launch": d_bytes, "us_per_launch": d_us, "gbs": d_gbs, "frac": d_gbs / peak,
                       "note": "delta-only launch (no base weight) over the same 3 experts / rows"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    line["config"]["rows_padded"] = rows
    line["config"]["num_ctas"] = ctas or "all SMs"  # launch width chosen by device.tune_num_ctas
    if rank == 0 and not args.no_cpu_baseline:
        dt, n = cpu_c1_baseline()
        line["cpu_baseline"] = {"value": C1_B / dt, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": f"{n} full C1 step(s): numpy x@W + x_g@reconstruct() per expert group"}
    return line


C4_T, C4_E = 2048, 16


def _c4_cpu(max_groups: int = 1):
    """Reference algorithm for one expert group of the prefill (x_g@W + x_g@reconstruct),
    timed and scaled to all groups (bounded sample)."""
    from paper_2406_09041_b200 import compress, synth
    rng = np.random.default_rng(0)
    W = rng.normal(0, 0.02, size=(C1_M, C1_N)).astype(np.float32)
    art = compress.deserialize_artifact(synth.synthetic_expert_artifact(1, [(C1_M, C1_N)], "e0"))
    layer = _oracle_layers([art])[0]
    x = rng.normal(0, 1, size=(C4_T // C4_E, C1_M)).astype(np.float32)
    t0 = time.perf_counter()
    for _ in range(max_groups):
        _ = x @ W + x @ layer.reconstruct()
    return (time.perf_counter() - t0) / max_groups * C4_E


def run_c4(args, ws, rank, local, ClockSampler, peaks):
    """C4: prefill of 2048 tokens (16 experts x 128) through one 4096x14336 fused linear:
    base GEMM and delta contraction on tcgen05 (one launch per expert group of 128 rows)."""
    import json
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, LinearPlan,
                                               pack_x)
    geom = LinearGeometry(C1_M, (C1_N,))
    g = torch.Generator(device="cuda").manual_seed(rank)
    dw = DeviceWeight.empty(geom)
    dw.load_block(0, (torch.randn((C1_M, C1_N), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
    table = ExpertTable("cuda")
    for e in range(C4_E):
        blob = synth.synthetic_expert_artifact(100 + e, [(C1_M, C1_N)], f"e{e}")
        table.set(e, DeviceDelta.from_blocks([compress.deserialize_artifact(blob).layers[0]], geom))
    per = C4_T // C4_E
    x = torch.randn((C4_T, C1_M), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.empty((C4_T, C1_N), dtype=torch.bfloat16, device="cuda")
    plans = [LinearPlan(pack_x(x[e * per:(e + 1) * per].contiguous()), per, dw, table, [(0, per, e)],
                        y[e * per:(e + 1) * per], geom=geom) for e in range(C4_E)]
    for _ in range(args.warmup):
        for p in plans:
            p()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    stream = torch.cuda.current_stream()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        st.record(stream)
        for _ in range(args.steps):
            for p in plans:
                p()
        en.record(stream)
        torch.cuda.synchronize()
    ms_t = torch.tensor([st.elapsed_time(en) / args.steps], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    flops = 2.0 * C4_T * C1_M * C1_N * 2  # base + delta contraction
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
        pk = json.load(f)
    peak = float(pk.get("bf16_tflops", 1590.0))
    achieved = flops / (ms / 1e3) / 1e12
    # e2e: host x (pinned) -> device, pack + fused launches, y -> host
    xh = x.cpu().pin_memory()
    yh = torch.empty((C4_T, C1_N), dtype=torch.bfloat16).pin_memory()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x.copy_(xh, non_blocking=True)
        for e, p in enumerate(plans):
            pack_x(x[e * per:(e + 1) * per].contiguous(), out=p.keep[0])  # canonical layout of the fresh input
            p()
        yh.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    line = {
        "metric": "prefill tokens/sec, one Mistral MLP linear 4096x14336, 2048 tokens over 16 experts",
        "value": ws * C4_T / (ms / 1e3), "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c4: prefill 2048 tokens x 16 experts (128 each), 4096x14336 fused linear",
                   "launches_per_step": C4_E},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": "measured burst",
                     "flops_per_step": flops, "kernel": "me_linear_tc_kernel<2>"},
        "e2e": {"value": ws * C4_T / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(xh.numel() * 2),
                "d2h_bytes_per_step": int(yh.numel() * 2)},
        "gpu_launches": C4_E * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        dt = _c4_cpu()
        line["cpu_baseline"] = {"value": C4_T / dt, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": "1 expert group of 128 tokens (x_g@W + x_g@reconstruct) timed, x16"}
    return line


def run_ours(args, ws, rank, local, ClockSampler, peaks):
    if args.config == "c4":
        return run_c4(args, ws, rank, local, ClockSampler, peaks)
    if args.config == "c1":
        return run_c1(args, ws, rank, local, ClockSampler, peaks)
    from bench_mistral import run_c2
    if args.config == "c5":  # BASELINE configs[4]: 64 experts sharded over the ranks, replicated base
        if 64 % ws:
            raise ValueError("c5 shards 64 experts: --gpus must divide 64")
        args.experts = 64 // ws
        args.batch = args.batch or 128
    return run_c2(args, ws, rank, local, ClockSampler, peaks)
