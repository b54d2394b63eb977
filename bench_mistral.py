"""C2/C3 workload for bench.py: Mistral-7B-shaped multi-expert decode.

GPU arm: full 32-layer stack, E synthetic experts (2-bit codes + 8 fp16 salient rows
on all 224 decoder linears), batch of B requests assigned round-robin to experts,
128-token synthetic prompt state (random KV), one step = one generated token per
request.  The step is a CUDA graph of libmesw.so kernels only.

CPU arm (cpu_baseline / --impl reference): the reference algorithm restated in
numpy (oracle port; the reference is Python and is absent on the GPU box): shared
base x@W for the batch, then per expert group x_g @ reconstruct() with the dense
delta cached (the reference's best case; as shipped it re-decodes every call),
plus RMSNorm / RoPE / attention / SwiGLU glue.  Timed on a bounded sample -- one
decoder layer -- and scaled to the 32-layer step (+ lm_head).
"""

from __future__ import annotations

import os
import time

import numpy as np

DEFAULT_B = 32
PROMPT = 128
CTX = 256


def _expert_names(E):
    base = ["instruct", "math", "code"]
    return [base[e] if e < 3 else f"expert{e}" for e in range(E)]


def build_engine(B, E, seed=0, n_layers=None, device="cuda", experts=None, requests=None):
    """Engine with the base (replicated) and experts `experts` (global ids; default
    0..E-1) resident; batch = `requests` (global expert id per request; default
    round-robin over the resident experts)."""
    from paper_2406_09041_b200 import compress, synth
    from paper_2406_09041_b200.mistral import MistralMultiExpert
    experts = list(range(E)) if experts is None else list(experts)
    shape = synth.MistralShape()
    eng = MistralMultiExpert(shape, max_batch=B + 16 * len(experts), ctx_max=CTX, device=device,
                             n_layers=n_layers)
    eng.wrap_positions = True  # steady-state benchmark: long runs wrap positions (never in serving)
    eng.load_synthetic_base(seed=seed)
    shapes = synth.mistral_expert_shapes(shape, eng.n_layers)
    names = _expert_names(max(experts) + 1)
    for e in experts:
        blob = synth.synthetic_expert_artifact(1000 + e, shapes, names[e])
        eng.add_expert(names[e], compress.deserialize_artifact(blob))
        del blob
    if requests is None:
        requests = [experts[t % len(experts)] for t in range(B)]
    eng.set_batch([names[e] for e in requests], [PROMPT] * len(requests))
    eng.fill_random_kv(PROMPT, seed=seed + 7)
    return eng


def run_c2(args, ws, rank, local, ClockSampler, peaks):
    import torch
    B = args.batch or DEFAULT_B
    E = args.experts
    # expert-sharded weak scaling: E experts per GPU (E*ws in total, expert e on rank e mod ws),
    # base replicated (seed 0 everywhere); rank 0 assigns B*ws requests round-robin over all
    # experts and dispatches each to its owner -- a host control message, no data collective
    from paper_2406_09041_b200.shard import Placement, dispatch
    pl = Placement(E * ws, ws)
    reqs = [(i, i % (E * ws), None) for i in range(B * ws)] if rank == 0 else None
    mine = dispatch(reqs, pl, rank) if ws > 1 else reqs
    eng = build_engine(B, E, seed=0, experts=pl.local_experts(rank), requests=[r[1] for r in mine])
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    R = eng.B  # engine rows (expert groups padded to 16-row boundaries)
    eng.ids[:R] = torch.randint(0, eng.shape.vocab, (R,), generator=g, device="cuda", dtype=torch.int32)
    eng.capture()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        eng.replay()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        st.record(stream)
        for _ in range(args.steps):
            eng.replay()
        en.record(stream)
        torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    ms_t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    per_step = ms / args.steps
    tok_s = ws * B * args.steps / (ms / 1e3)
    nbytes = eng.bytes_per_step()

    # dominant kernel: the fused multi-expert linear.  Time all linear launches of a step
    # (4 per layer + lm_head) alone, CUDA events on the launching stream.
    lin_graph = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    n_lin = 0
    with torch.cuda.stream(s2):
        lin_graph.capture_begin()
        for (_, _, _, layers, head) in eng._plans:
            for layer_plans in layers:
                for p in layer_plans:
                    p(s2)
                    n_lin += 1
            head(s2)
            n_lin += 1
        lin_graph.capture_end()
    torch.cuda.current_stream().wait_stream(s2)
    for _ in range(3):
        lin_graph.replay()
    torch.cuda.synchronize()
    st.record(stream)
    for _ in range(args.steps):
        lin_graph.replay()
    en.record(stream)
    torch.cuda.synchronize()
    lin_ms = st.elapsed_time(en) / args.steps
    lin_bytes = nbytes["linears"] + nbytes["head"]
    peak, peak_kind = peaks()
    achieved = lin_bytes / (lin_ms / 1e3) / 1e9
    delta_gbs = nbytes["delta"] / (lin_ms / 1e3) / 1e9 * (nbytes["delta"] / max(nbytes["delta"], 1))

    # e2e through the public API: pinned host ids -> device -> graph step -> next ids -> host
    host_in = torch.zeros(R, dtype=torch.int32).pin_memory()
    host_out = torch.zeros(R, dtype=torch.int32).pin_memory()
    host_in.copy_(eng.ids[:R].cpu())
    for _ in range(args.warmup):
        eng.decode(host_in, host_out)
        host_in.copy_(host_out)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        eng.decode(host_in, host_out)
        host_in.copy_(host_out)
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_t = torch.tensor([e2e_s], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())

    traffic = None
    try:
        import json
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            tr = json.load(f).get(f"c2_B{B}_E{E}")
            traffic = tr["traffic"] if tr else None  # dram bytes of one step's linear launches
    except Exception:
        pass

    line = {
        "metric": "decode tokens/sec with N mixed experts (Mistral-7B shape); delta-GEMM HBM GB/s",
        "value": tok_s, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init Mistral-7B-shaped base, synthetic 2-bit deltas)",
        "config": {"workload": (f"c5: 64 experts sharded over {ws} GPU(s), " if getattr(args, "config", "c2") == "c5" else "c2: ")
                               + f"full Mistral-7B decoder stack (32 layers), {E} experts per GPU "
                               f"(b=2 codes + 8 fp16 salient rows on all 224 decoder linears), "
                               f"batch {B} mixed decode, ctx {PROMPT}+",
                   "batch": B, "experts": E, "l2": f"per-step weights {nbytes['total']/1e9:.1f} GB >> 126 MB L2",
                   "parallelism": f"expert-sharded replicas x{ws} (replicated base, no collective)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": f"me_linear_tc_kernel<2, true> (all {n_lin} fused linear launches of a step)",
                     "bytes_per_step": lin_bytes, "kernel_ms_per_step": lin_ms,
                     "kernel_share_of_step": lin_ms / per_step},
        "delta_gemm": {"bytes_per_step": nbytes["delta"],
                       "note": "delta bytes (codes+salient+steps) streamed by the fused linears"},
        "e2e": {"value": ws * B / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": 4 * R,
                "d2h_bytes_per_step": 4 * R},
        "gpu_launches": eng.launches_per_step() * args.steps,
        "clocks": clk.summary(),
        "step_bytes": nbytes,
    }
    if rank == 0 and not args.no_cpu_baseline:
        del eng, lin_graph
        torch.cuda.empty_cache()
        cpu = cpu_layer_sample(B, E, reps=1)
        line["cpu_baseline"] = cpu
    return line


# ------------------------------------------------------------------------- CPU arm

class _CpuLayer:
    """One Mistral decoder layer on the host, reference-style numpy (f32)."""

    def __init__(self, B, E, seed=0):
        from oracle import mesw as om
        from paper_2406_09041_b200 import compress, synth
        self.shape = s = synth.MistralShape()
        rng = np.random.default_rng(seed)
        kv = s.n_kv_heads * s.head_dim
        self.dims = {"q": (s.hidden, s.hidden), "k": (s.hidden, kv), "v": (s.hidden, kv), "o": (s.hidden, s.hidden),
                     "gate": (s.hidden, s.intermediate), "up": (s.hidden, s.intermediate),
                     "down": (s.intermediate, s.hidden)}
        self.W = {n: (rng.standard_normal(size=d, dtype=np.float32) * 0.02) for n, d in self.dims.items()}
        self.norm = np.ones(s.hidden, np.float32)
        shapes = [self.dims[n] for n in ("q", "k", "v", "o", "gate", "up", "down")]
        self.layers = []  # per expert: dict proj -> oracle layer
        for e in range(E):
            blob = synth.synthetic_expert_artifact(1000 + e, shapes, f"e{e}")
            _, ls = om.parse_artifact(blob)
            self.layers.append(dict(zip(("q", "k", "v", "o", "gate", "up", "down"), ls)))
        self.dense = None
        self.B, self.E = B, E
        self.kc = rng.standard_normal(size=(B, PROMPT + 1, s.n_kv_heads, s.head_dim), dtype=np.float32)
        self.vc = rng.standard_normal(size=(B, PROMPT + 1, s.n_kv_heads, s.head_dim), dtype=np.float32)
        self.h = rng.standard_normal(size=(B, s.hidden), dtype=np.float32)
        self.groups = [np.arange(B)[np.arange(B) % E == e] for e in range(E)]

    def cache_dense(self):
        self.dense = [{n: L.reconstruct() for n, L in per.items()} for per in self.layers]

    def _lin(self, x, name, cached=True):
        y = x @ self.W[name]
        for e, idx in enumerate(self.groups):
            if idx.size:
                d = self.dense[e][name] if cached else self.layers[e][name].reconstruct()
                y[idx] += x[idx] @ d
        return y

    def step(self, cached=True):
        s = self.shape
        h = self.h

        def rms(x):
            return x / np.sqrt((x * x).mean(-1, keepdims=True) + s.rms_eps) * self.norm

        x = rms(h)
        q = self._lin(x, "q", cached).reshape(self.B, s.n_heads, s.head_dim)
        k = self._lin(x, "k", cached).reshape(self.B, s.n_kv_heads, s.head_dim)
        v = self._lin(x, "v", cached).reshape(self.B, s.n_kv_heads, s.head_dim)
        half = s.head_dim // 2
        ang = PROMPT * (s.rope_theta ** (-2.0 * np.arange(half) / s.head_dim))
        c, sn = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)

        def rope(t):
            a, b = t[..., :half], t[..., half:]
            return np.concatenate([a * c - b * sn, b * c + a * sn], -1)

        q, k = rope(q), rope(k)
        self.kc[:, PROMPT] = k
        self.vc[:, PROMPT] = v
        G = s.n_heads // s.n_kv_heads
        qg = q.reshape(self.B, s.n_kv_heads, G, s.head_dim)
        sc = np.einsum("bkgd,btkd->bkgt", qg, self.kc) / np.sqrt(s.head_dim)
        sc = np.exp(sc - sc.max(-1, keepdims=True))
        sc /= sc.sum(-1, keepdims=True)
        att = np.einsum("bkgt,btkd->bkgd", sc, self.vc).reshape(self.B, -1)
        h = h + self._lin(att.astype(np.float32), "o", cached)
        x = rms(h)
        gt = self._lin(x, "gate", cached)
        up = self._lin(x, "up", cached)
        h = h + self._lin((gt / (1 + np.exp(-gt)) * up).astype(np.float32), "down", cached)
        return h


def _head_time(B):
    from paper_2406_09041_b200 import synth
    s = synth.MistralShape()
    rng = np.random.default_rng(0)
    Wh = rng.standard_normal(size=(s.hidden, s.vocab), dtype=np.float32) * 0.02
    x = rng.standard_normal(size=(B, s.hidden), dtype=np.float32)
    t0 = time.perf_counter()
    np.argmax(x @ Wh, -1)
    return time.perf_counter() - t0


def cpu_layer_sample(B, E, reps=1):
    layer = _CpuLayer(B, E)
    layer.cache_dense()
    layer.step()
    t0 = time.perf_counter()
    for _ in range(reps):
        layer.step()
    t_layer = (time.perf_counter() - t0) / reps
    t_step = 32 * t_layer + _head_time(B)
    return {"value": B / t_step, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{reps} x one decoder layer (7 projections, B={B}, {E} experts, dense deltas cached = "
                      f"reference best case) timed, scaled x32 layers + lm_head; numpy/OpenBLAS all threads",
            "layer_s": t_layer}


def _time_layer(layer, steps, warmup):
    for _ in range(warmup):
        layer.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        layer.step()
    return (time.perf_counter() - t0) / steps


def reference_arm_c2(args):
    ws = args.gpus
    c5 = getattr(args, "config", "c2") == "c5"
    if c5:  # the rank-0 share of 64 sharded experts, batch 128 per GPU (as the GPU arm)
        args.experts = 64 // ws
        args.batch = args.batch or 128
    B = args.batch or DEFAULT_B
    E = args.experts
    # at many experts the cached dense deltas do not fit host memory (0.87 GB f32 per expert
    # and layer): time a 4-expert sample and scale its delta part to E experts
    E_s = min(E, 4)
    layer = _CpuLayer(B, E_s)
    layer.cache_dense()
    t_layer = _time_layer(layer, args.steps, args.warmup)
    sample = f"each step = one decoder layer (B={B}, {E} experts, cached dense deltas) scaled x32 + lm_head"
    if E_s < E:
        groups, layer.groups = layer.groups, []
        t_base = _time_layer(layer, args.steps, 1)
        layer.groups = groups
        t_layer = t_base + (E / E_s) * (t_layer - t_base)
        sample = (f"one decoder layer, B={B}: base part timed, delta part timed on {E_s} of {E} experts "
                  f"(cached dense deltas) and scaled x{E / E_s:g}; x32 layers + lm_head")
    t_step = 32 * t_layer + _head_time(B)
    val = B / t_step
    return {"impl": "reference", "metric": "decode tokens/sec with N mixed experts (Mistral-7B shape); "
                                          "delta-GEMM HBM GB/s",
            "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"c5: 64 experts sharded over {ws} GPU(s), " if getattr(args, "config", "c2") == "c5" else "c2: ")
                               + f"full Mistral-7B decoder stack (32 layers), {E} experts per GPU "
                                   f"(b=2 codes + 8 fp16 salient rows on all 224 decoder linears), "
                                   f"batch {B} mixed decode, ctx {PROMPT}+", "batch": B, "experts": E},
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
