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
        dts = [_c4_cpu() * _C4_SCALE for _ in range(args.steps)]
        val = C4_T / (sum(dts) / len(dts))
        return {"impl": "reference", "metric": "prefill tokens/sec through a Mistral decoder layer's 4 fused linears, 2048 tokens over 16 experts",
                "value": val, "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * C4_T / val, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": "c4: prefill 2048 tokens x 16 experts (128 each) through q|k|v, o, gate|up, down"},
                "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port",
                                 "sample": "per step: 1 expert group of 128 tokens (x_g@W + x_g@reconstruct) of a "
                                           "4096x14336 linear, x16 groups, scaled by the 4 linears' flops"},
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

    # e2e through the public API: every step copies its own input from pinned host memory,
    # runs me_linear (device-side expert grouping, caller row order) and reads its result back
    # into pinned host memory, and the host waits for that result.  Two steps are in flight
    # (a serving loop's double buffering): step i+1's upload and launch are queued before the
    # host waits for step i, and copies run on their own streams so they overlap the kernel.
    from paper_2406_09041_b200.device import MeLinearGraph
    xh = [torch.from_numpy(x_np[order]).to(torch.bfloat16).pin_memory() for _ in range(2)]
    yh = [torch.empty((C1_B, C1_N), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    yd = [torch.empty((C1_B, C1_N), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    s_in, s_out, s_k = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
    done = [torch.cuda.Event() for _ in range(2)]
    # one captured me_linear per (buffer, weight replica): a serving loop replays the call
    graphs = {(b, r): MeLinearGraph(xd[b], sets[r][0], sets[r][1], segs, yd[b], offset_codes=True,
                                    num_ctas=ctas) for b in range(2) for r in range(replicas)}

    def e2e_step(i):
        b = i % 2
        with torch.cuda.stream(s_in):
            s_in.wait_event(done[b])  # buffer b's previous use fully read back
            xd[b].copy_(xh[b], non_blocking=True)
            up = torch.cuda.Event()
            up.record(s_in)
        s_k.wait_event(up)
        graphs[(b, i % replicas)]()
        comp = torch.cuda.Event()
        comp.record(s_k)
        with torch.cuda.stream(s_out):
            s_out.wait_event(comp)
            yh[b].copy_(yd[b], non_blocking=True)
            done[b].record(s_out)
        if i >= 1:
            done[(i - 1) % 2].synchronize()  # the host has step i-1's result

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    done[(args.steps - 1) % 2].synchronize()
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
        "e2e": {"value": ws * C1_B / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(xh[0].numel() * 2),
                "d2h_bytes_per_step": int(yh[0].numel() * 2),
                "path": "device.MeLinearGraph (me_linear captured once: device-side grouping, y_rows "
                        "epilogue), pinned H2D/D2H every step, 2 steps in flight on separate copy streams"},
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


C4_KINDS = (("qkv", 4096, (4096, 1024, 1024)), ("o", 4096, (4096,)), ("gate_up", 4096, (14336, 14336)),
            ("down", 14336, (4096,)))


def run_c4(args, ws, rank, local, ClockSampler, peaks):
    """C4: prefill of 2048 tokens over 16 experts (128 tokens each) through the 4 fused linears
    of a Mistral decoder layer (q|k|v, o, gate|up, down) with the K3 prefill kernel: the delta
    is folded into the tcgen05 A operand, so the tensor work is the base GEMM's.  One step =
    the 4 launches; 2 rotating weight/expert replicas (L2-cold weights)."""
    import json
    import torch
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, PrefillPlan,
                                               pack_x)
    g = torch.Generator(device="cuda").manual_seed(rank)
    groups = C4_T // 128
    slots = [gi * C4_E // groups for gi in range(groups)]
    reps = 2
    kinds = []
    for name, m, blocks in C4_KINDS:
        geom = LinearGeometry(m, blocks)
        x = torch.randn((C4_T, m), generator=g, device="cuda").to(torch.bfloat16)
        xc = pack_x(x)
        y = torch.empty((C4_T, geom.n), dtype=torch.bfloat16, device="cuda")
        fused, base = [], []
        for r in range(reps):
            dw = DeviceWeight.empty(geom)
            for bi, nb in enumerate(blocks):
                dw.load_block(bi, (torch.randn((m, nb), generator=g, device="cuda") * 0.02).to(torch.bfloat16))
            table = ExpertTable("cuda")
            for e in range(C4_E):
                blob = synth.synthetic_expert_artifact(100 * r + e, [(m, nb) for nb in blocks], f"e{e}")
                table.set(e, DeviceDelta.from_blocks(compress.deserialize_artifact(blob).layers, geom))
                del blob
            fused.append(PrefillPlan(xc, C4_T, C4_T, dw, table, slots, y))
            base.append(PrefillPlan(xc, C4_T, C4_T, dw, None, [-1] * groups, y))
        kinds.append((name, m, sum(blocks), fused, base, x))

    def run_all(which, i):
        for k in kinds:
            k[3 if which == "fused" else 4][i % reps]()

    def timed(which, steps, clk=None):
        for i in range(args.warmup):
            run_all(which, i)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for i in range(steps):
            run_all(which, i)
        en.record()
        torch.cuda.synchronize()
        return st.elapsed_time(en) / steps

    with ClockSampler(local) as clk:
        ms = timed("fused", args.steps)
    ms_base = timed("base", args.steps)
    per_kind = {}
    for name, m, n, fused, base, _ in kinds:  # per-kind time of the fused launch
        for i in range(3):
            fused[i % reps]()
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for i in range(args.steps):
            fused[i % reps]()
        en.record()
        torch.cuda.synchronize()
        t = st.elapsed_time(en) / args.steps
        per_kind[name] = {"ms": t, "tflops": 2.0 * C4_T * m * n / (t / 1e3) / 1e12}
    ms_t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    flops = sum(2.0 * C4_T * m * n for _, m, n, _, _, _ in kinds)  # base GEMM flops of the 4 linears
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
        pk = json.load(f)
    peak = float(pk.get("bf16_tflops", 1590.0))
    achieved = flops / (ms / 1e3) / 1e12
    for v in per_kind.values():
        v["frac"] = v["tflops"] / peak
    # e2e through the public API: host x (pinned) -> device -> canonical layout -> 4 launches -> y -> host
    xh = [k[5].cpu().pin_memory() for k in kinds]
    yh = [torch.empty((C4_T, k[2]), dtype=torch.bfloat16).pin_memory() for k in kinds]
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        for (name, m, n, fused, base, x), h, yo in zip(kinds, xh, yh):
            x.copy_(h, non_blocking=True)
            p = fused[i % reps]
            pack_x(x, out=p.keep[0])
            p()
            yo.copy_(p.keep[3][:, :n], non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    line = {
        "metric": "prefill tokens/sec through a Mistral decoder layer's 4 fused linears, 2048 tokens over 16 experts",
        "value": ws * C4_T / (ms / 1e3), "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c4: prefill 2048 tokens x 16 experts (128 each) through q|k|v, o, gate|up, down "
                               "(one decoder layer's fused linears, K3 kernel)", "launches_per_step": len(kinds),
                   "l2": "2 rotating weight/expert replicas per linear (> 126 MB L2)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": "measured burst (bf16_tflops)",
                     "flops_per_step": flops, "flops_note": "base GEMM flops; the delta is folded into the A "
                                                           "operand and adds no tensor flops",
                     "base_only_ms": ms_base, "base_only_frac": flops / (ms_base / 1e3) / 1e12 / peak,
                     "per_kind": per_kind, "kernel": "me_linear_prefill_kernel (K3)"},
        "e2e": {"value": ws * C4_T / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": int(sum(h.numel() * 2 for h in xh)),
                "d2h_bytes_per_step": int(sum(v.numel() * 2 for v in yh))},
        "gpu_launches": len(kinds) * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        dt = _c4_cpu() * _C4_SCALE
        line["cpu_baseline"] = {"value": C4_T / dt, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": "1 expert group of 128 tokens (x_g@W + x_g@reconstruct) of a 4096x14336 "
                                          "linear timed, x16 groups, scaled by the 4 linears' flops"}
    return line


_C4_SCALE = sum(m * sum(b) for _, m, b in C4_KINDS) / (C1_M * C1_N)  # 4 layer linears vs one 4096x14336


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
