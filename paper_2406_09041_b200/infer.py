"""Serving-time API: delta providers, delta_matvec, the batched multi-model forward
and bench_decode -- the SPEC `infer` module, which the
reference describes but does not ship, built on the fused GPU kernel.

`GpuCompressedProvider` satisfies the reference's duck-typed provider protocol
(toylm.py:171-186): `matvec_batch`, `matvec`, `rows`, `row` are METHODS (the
reference's own CompressedDelta cannot be a provider because its `rows` is an
int property, compress.py:96-98).  It takes/returns float32 numpy arrays and runs
every product on the GPU.  Float32 inputs are split into bf16 hi + lo halves
that the kernel contracts as two token rows, so the delta term is accurate to
~2^-16 relative (the kernel's own codes, steps and fp16 rows are exact).
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np
import torch

from .compress import CompressedDelta
from .device import DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, me_linear

__all__ = [
    "base_digest",
    "GpuCompressedProvider",
    "ExactProvider",
    "LowRankProvider",
    "ZeroProvider",
    "delta_matvec",
    "BatchPlan",
    "ToyBase",
    "batched_multi_model_forward",
    "batched_greedy_decode",
    "bench_decode",
    "split_bf16",
]

_MAX_ROWS = 32  # hi/lo token pairs per launch (kernel handles <= 64 tokens)


def base_digest(model) -> str:
    """toylm.base_digest (toylm.py:115-120): SHA-256 over the little-endian f32 bytes of the
    base matrices in `weight_matrices()` order (embedding, hidden layers..., head) -- the
    identity an expert artifact's manifest binds to.  Host-side, computed once at load.
    `model`: anything with weight_matrices(), or an iterable of matrices."""
    import hashlib
    mats = model.weight_matrices() if hasattr(model, "weight_matrices") else model
    h = hashlib.sha256()
    for w in mats:
        if hasattr(w, "detach"):
            w = w.detach().float().cpu().numpy()
        h.update(np.ascontiguousarray(w, dtype="<f4").tobytes())
    return h.hexdigest()

def split_bf16(x: torch.Tensor, m_pad: int) -> torch.Tensor:
    """f32 [T, m] -> bf16 [2T, m_pad]: rows 0..T-1 = bf16(x), rows T.. = bf16(x - hi)."""
    T, m = x.shape
    out = torch.zeros((2 * T, m_pad), dtype=torch.bfloat16, device=x.device)
    hi = x.to(torch.bfloat16)
    out[:T, :m] = hi
    out[T:, :m] = (x - hi.to(torch.float32)).to(torch.bfloat16)
    return out


class GpuCompressedProvider:
    """Compressed delta of one layer, resident on the GPU (SPEC DeltaProvider `Compressed`)."""

    def __init__(self, layer: CompressedDelta, device="cuda"):
        self.device = torch.device(device)
        self.delta = DeviceDelta.from_blocks([layer], device=self.device)
        self.table = ExpertTable(self.device, capacity=1)
        self.table.set(0, self.delta)
        self.geom = self.delta.geom

    @property
    def shape(self) -> tuple:
        return (self.geom.m, self.geom.n)

    def _run(self, h: torch.Tensor) -> torch.Tensor:
        T = h.shape[0]
        outs = []
        for s in range(0, T, _MAX_ROWS):
            part = h[s:s + _MAX_ROWS]
            t = part.shape[0]
            x2 = split_bf16(part, self.geom.m_pad)
            y2 = me_linear(x2, None, self.table, [(0, 2 * t, 0)], out_dtype=torch.float32, geom=self.geom)
            outs.append(y2[:t] + y2[t:])
        return torch.cat(outs, 0) if outs else torch.zeros((0, self.geom.n), device=self.device)

    def matvec_batch(self, h) -> np.ndarray:
        """f32 [T, m] -> f32 [T, n] = h . reconstruct() without materialising it."""
        h = np.asarray(h, dtype=np.float32)
        if h.ndim != 2 or h.shape[1] != self.geom.m:
            raise ValueError(f"expected input of shape (T, {self.geom.m}), got {h.shape}")
        ht = torch.from_numpy(np.ascontiguousarray(h)).to(self.device)
        return self._run(ht).cpu().numpy()

    def matvec(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float32)
        if x.ndim != 1:
            raise ValueError("matvec expects a 1-D vector")
        return self.matvec_batch(x[None, :])[0]

    def rows(self, ids) -> np.ndarray:
        """Delta rows reconstruct()[ids] (embedding layer), bit-exact: one-hot inputs."""
        ids = np.asarray(ids, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= self.geom.m):
            raise ValueError("row id out of range")
        onehot = torch.zeros((ids.size, self.geom.m), dtype=torch.float32, device=self.device)
        if ids.size:
            onehot[torch.arange(ids.size, device=self.device), torch.from_numpy(ids).to(self.device)] = 1.0
        return self._run(onehot).cpu().numpy()

    def row(self, i) -> np.ndarray:
        return self.rows(np.asarray([int(i)]))[0]


class ExactProvider:
    """SPEC `Exact(DenseMatrix)`: plain f32 product (library GEMM, not the hot path)."""

    def __init__(self, dense, device="cuda"):
        self.d = torch.as_tensor(np.asarray(dense, np.float32)).to(device)

    def matvec_batch(self, h):
        return (torch.as_tensor(np.asarray(h, np.float32)).to(self.d.device) @ self.d).cpu().numpy()

    def matvec(self, x):
        return self.matvec_batch(np.asarray(x, np.float32)[None])[0]

    def rows(self, ids):
        return self.d[torch.as_tensor(np.asarray(ids, np.int64)).to(self.d.device)].cpu().numpy()

    def row(self, i):
        return self.rows([int(i)])[0]


class LowRankProvider(ExactProvider):
    """SPEC `LowRank`: (x.A).B."""

    def __init__(self, a, b, device="cuda"):
        self.a = torch.as_tensor(np.asarray(a, np.float32)).to(device)
        self.b = torch.as_tensor(np.asarray(b, np.float32)).to(device)
        self.d = None

    def matvec_batch(self, h):
        x = torch.as_tensor(np.asarray(h, np.float32)).to(self.a.device)
        return ((x @ self.a) @ self.b).cpu().numpy()

    def rows(self, ids):
        return (self.a[torch.as_tensor(np.asarray(ids, np.int64)).to(self.a.device)] @ self.b).cpu().numpy()


class ZeroProvider:
    """SPEC `Zero`."""

    def __init__(self, shape):
        self.shape = tuple(shape)

    def matvec_batch(self, h):
        return np.zeros((np.asarray(h).shape[0], self.shape[1]), np.float32)

    def matvec(self, x):
        return np.zeros(self.shape[1], np.float32)

    def rows(self, ids):
        return np.zeros((len(ids), self.shape[1]), np.float32)

    def row(self, i):
        return np.zeros(self.shape[1], np.float32)


def delta_matvec(x, p) -> np.ndarray:
    """y = x . Dtilde for any provider (Compressed runs the fused GPU kernel)."""
    x = np.asarray(x, dtype=np.float32)
    if p is None:
        raise ValueError("provider is None")
    return np.asarray(p.matvec(x), np.float32)


# --------------------------------------------------------------------------- toy batched forward

@dataclass(frozen=True)
class BatchPlan:
    """queries (query id, expert id, token sequence)."""

    queries: tuple

    @classmethod
    def of(cls, items) -> "BatchPlan":
        return cls(tuple((q, e, tuple(int(t) for t in toks)) for q, e, toks in items))


def _positional_bias(n: int, width: int) -> np.ndarray:
    """Sinusoidal positional table of the toy model (toylm.py:87-93)."""
    pos = np.arange(n, dtype=np.float64)[:, None]
    dim = np.arange(width, dtype=np.float64)[None, :]
    angle = pos / np.power(10000.0, (2.0 * (dim // 2)) / width)
    return np.where(dim % 2 == 0, np.sin(angle), np.cos(angle)).astype(np.float32)


class ToyBase:
    """The reference toy model's base weights resident on the GPU.

    Layer order follows toylm.ToyLM.weight_matrices (embedding, hidden..., head).
    Each f32 weight is held as a bf16 pair W = W_hi + W_lo (fragment layout), so the
    fused kernel reproduces f32 products to ~2^-16 relative (SPEC.md:438 asks 1e-4).
    """

    def __init__(self, embedding, layers, head, device="cuda"):
        self.device = torch.device(device)
        self.embedding = torch.as_tensor(np.asarray(embedding, np.float32)).to(self.device)
        self.vocab, self.width = self.embedding.shape
        self.layers = [self._pair(w) for w in layers]
        self.head = self._pair(head)
        self.depth = len(self.layers)

    def _pair(self, w):
        wf = torch.as_tensor(np.asarray(w, np.float32)).to(self.device)
        hi = wf.to(torch.bfloat16)
        lo = (wf - hi.to(torch.float32)).to(torch.bfloat16)
        return DeviceWeight.from_dense([hi], self.device), DeviceWeight.from_dense([lo], self.device)

    @classmethod
    def from_model(cls, model, device="cuda") -> "ToyBase":
        return cls(model.embedding, model.layers, model.head, device)

    @property
    def n_weight_layers(self) -> int:
        return self.depth + 2


class ExpertSet:
    """Resident experts of a toy model: one ExpertTable per weight layer."""

    def __init__(self, base: ToyBase):
        self.base = base
        self.tables = [ExpertTable(base.device) for _ in range(base.n_weight_layers)]
        self.slots: dict = {}

    def add(self, expert_id, artifact) -> int:
        layers = artifact.layers if hasattr(artifact, "layers") else list(artifact)
        if len(layers) != self.base.n_weight_layers:
            raise ValueError("artifact layer count does not match the base model")
        return self.add_device(expert_id, [DeviceDelta.from_blocks([layer], device=self.base.device)
                                           for layer in layers])

    def add_device(self, expert_id, deltas: list) -> int:
        """Install already-resident per-layer DeviceDeltas (e.g. a registry handle's)."""
        if len(deltas) != self.base.n_weight_layers:
            raise ValueError("artifact layer count does not match the base model")
        slot = len(self.slots)
        for t, d in zip(self.tables, deltas):
            t.set(slot, d)
        self.slots[expert_id] = slot
        return slot


_CHUNK = 32  # positions per launch group (hi + lo rows <= 64 tokens)


def _precise_linear(x: torch.Tensor, pair, table: ExpertTable, segs) -> torch.Tensor:
    """f32 x [c, m] -> f32 x.(W_hi + W_lo) + x.Dtilde_{expert}: two fused launches.
    Launch 1 contracts [x_hi; x_lo] with W_hi and the expert deltas; launch 2 adds x_hi.W_lo."""
    w_hi, w_lo = pair
    c = x.shape[0]
    x2 = split_bf16(x, w_hi.geom.m_pad)
    segs2 = segs + [(b + c, e + c, sl) for b, e, sl in segs]
    y2 = me_linear(x2, w_hi, table if segs else None, segs2, out_dtype=torch.float32)
    y3 = me_linear(x2[:c], w_lo, None, [], out_dtype=torch.float32)
    return y2[:c] + y2[c:] + y3


def batched_multi_model_forward(base: ToyBase, registry, plan) -> list:
    """SPEC.md:433-438 on the GPU: shared-base x.W and every expert group's delta in
    fused launches per layer; per-query results in input order.

    `registry` is the SPEC's registry handle (`registry.ExpertRegistry` whose loader returns
    per-layer device deltas, e.g. `registry.GpuExpert`): every distinct expert of the plan
    is acquired (loaded on demand, pinned) for the duration of the batch and released
    afterwards with a fence on the stream that ran it.  An
    `ExpertSet` of already-resident experts is accepted too.

    Returns [(query_id, logits f32 [len, V] or None, error or None)].  An unknown
    expert (or one that cannot be made resident) yields an error entry for that query
    and the batch continues.
    """
    queries = plan.queries if isinstance(plan, BatchPlan) else tuple(plan)
    if isinstance(registry, ExpertSet):
        return _forward_resident(base, registry, queries)
    from .errors import RegistryError
    acquired, failed = [], {}
    experts = ExpertSet(base)
    try:
        for eid in dict.fromkeys(q[1] for q in queries):  # distinct, first-seen order
            try:
                handle = registry.acquire(eid)
            except RegistryError as e:  # UnknownExpertError, BudgetExceededError
                failed[eid] = f"{type(e).__name__}: {e}"
                continue
            acquired.append(eid)
            experts.add_device(eid, list(handle.layers))
        res = _forward_resident(base, experts, queries)
    finally:
        stream = torch.cuda.current_stream(base.device)
        for eid in acquired:
            registry.release(eid, stream)
    return [(qid, None, failed[queries[i][1]]) if queries[i][1] in failed else (qid, lg, err)
            for i, (qid, lg, err) in enumerate(res)]


def _forward_resident(base: ToyBase, experts: ExpertSet, queries, pos0=None) -> list:
    """pos0[qi]: position of query qi's first token (default 0; decode steps use the last
    position only -- the toy model has no attention, toylm.py:214-248)."""
    results = {}
    order = []
    for qi, (qid, eid, toks) in enumerate(queries):
        if eid not in experts.slots:
            results[qi] = (qid, None, f"unknown expert {eid!r}")
        elif len(toks) == 0:
            results[qi] = (qid, None, "empty token sequence")
        else:
            order.append(qi)
    # group the valid queries by expert slot (stable), concatenate their positions
    order.sort(key=lambda qi: experts.slots[queries[qi][1]])
    dev = base.device
    ids, pos, spans, segs = [], [], {}, []
    cur = 0
    for qi in order:
        toks = np.asarray(queries[qi][2], np.int64)
        if toks.min() < 0 or toks.max() >= base.vocab:
            results[qi] = (queries[qi][0], None, "token id out of range")
            continue
        slot = experts.slots[queries[qi][1]]
        spans[qi] = (cur, cur + toks.size)
        if segs and segs[-1][2] == slot and segs[-1][1] == cur:
            segs[-1] = (segs[-1][0], cur + toks.size, slot)
        else:
            segs.append((cur, cur + toks.size, slot))
        ids.append(toks)
        pos.append(np.arange(toks.size) + (0 if pos0 is None else int(pos0[qi])))
        cur += toks.size
    if cur:
        all_ids = torch.from_numpy(np.concatenate(ids)).to(dev)
        pb = torch.from_numpy(_positional_bias(max(int(p.max()) for p in pos) + 1, base.width)).to(dev)
        h = base.embedding[all_ids] + pb[torch.from_numpy(np.concatenate(pos)).to(dev)]
        logits = torch.empty((cur, base.vocab), dtype=torch.float32, device=dev)
        emb_geom = LinearGeometry(base.vocab, (base.width,))
        for c0 in range(0, cur, _CHUNK):
            c1 = min(cur, c0 + _CHUNK)
            csegs = _clip_segments(segs, c0, c1)
            # embedding delta rows: one-hot inputs through the fused kernel (exact rows of reconstruct())
            onehot = torch.zeros((c1 - c0, _pad128(base.vocab)), dtype=torch.bfloat16, device=dev)
            onehot[torch.arange(c1 - c0, device=dev), all_ids[c0:c1]] = 1.0
            emb_delta = me_linear(onehot, None, experts.tables[0], csegs, out_dtype=torch.float32, geom=emb_geom)
            x = h[c0:c1] + emb_delta
            for li, pair in enumerate(base.layers):
                x = torch.clamp_min(_precise_linear(x, pair, experts.tables[1 + li], csegs), 0.0)
            logits[c0:c1] = _precise_linear(x, base.head, experts.tables[-1], csegs)
        out_np = logits.cpu().numpy()
        for qi, (a, b) in spans.items():
            results[qi] = (queries[qi][0], out_np[a:b].copy(), None)
    return [results[i] for i in range(len(queries))]


def _pad128(v: int) -> int:
    return (v + 127) // 128 * 128


def _pad_cols(x: torch.Tensor, width: int) -> torch.Tensor:
    if x.shape[1] == width:
        return x.contiguous()
    out = torch.zeros((x.shape[0], width), dtype=x.dtype, device=x.device)
    out[:, :x.shape[1]] = x
    return out


def _clip_segments(segs, c0: int, c1: int) -> list:
    out = []
    for b, e, s in segs:
        b2, e2 = max(b, c0), min(e, c1)
        if b2 < e2:
            out.append((b2 - c0, e2 - c0, s))
    return out


def batched_greedy_decode(base: ToyBase, registry, requests) -> list:
    """Greedy continuation for a batch of requests on the GPU, each with its own expert:
    requests = [(request id, expert id, prompt token ids, max_new)].  Equal to the reference's
    greedy_decode(base, providers_e, prompt, max_new) per request (toylm.py:234-248: one
    position per step, first-maximum argmax); every step is ONE batched multi-expert forward
    over all still-active requests.  `registry` as in
    batched_multi_model_forward (experts acquired for the whole decode, released after).
    Returns [(request id, token ids incl. the prompt, or None, error or None)]."""
    from .errors import RegistryError
    reqs = list(requests)
    own = not isinstance(registry, ExpertSet)
    experts = registry if not own else ExpertSet(base)
    acquired, failed = [], {}
    out = {}
    try:
        if own:
            for eid in dict.fromkeys(r[1] for r in reqs):
                try:
                    handle = registry.acquire(eid)
                except RegistryError as e:
                    failed[eid] = f"{type(e).__name__}: {e}"
                    continue
                acquired.append(eid)
                experts.add_device(eid, list(handle.layers))
        seqs = {}
        for rid, eid, prompt, max_new in reqs:
            if eid in failed:
                out[rid] = (rid, None, failed[eid])
            elif len(prompt) == 0:
                out[rid] = (rid, None, "empty prompt")
            else:
                seqs[rid] = [list(int(t) for t in prompt), int(max_new), eid]
        step = 0
        while True:
            active = [(rid, s) for rid, s in seqs.items() if step < s[1]]  # tokens generated so far = step
            if not active:
                break
            queries = [(rid, s[2], [s[0][-1]]) for rid, s in active]
            res = _forward_resident(base, experts, queries, pos0=[len(s[0]) - 1 for _, s in active])
            for (rid, s), (_, logits, err) in zip(active, res):
                if err is not None:
                    out[rid] = (rid, None, err)
                    del seqs[rid]
                else:
                    s[0].append(int(np.argmax(logits[-1])))
            step += 1
        for rid, s in seqs.items():
            out[rid] = (rid, s[0], None)
    finally:
        if own:
            stream = torch.cuda.current_stream(base.device)
            for eid in acquired:
                registry.release(eid, stream)
    return [out[r[0]] for r in reqs]


# --------------------------------------------------------------------------- bench_decode

def bench_decode(weight: DeviceWeight, table: ExpertTable, segments, x: torch.Tensor,
                 repetitions: int = 20, warmup: int = 3) -> dict:
    """SPEC.md:439-443 (Appendix F decomposition) for one multi-expert linear:
    base GEMV alone, delta stage alone, and the fused kernel; CUDA-event timed,
    first `warmup` reps dropped, median and p90 in milliseconds."""

    def timeit(fn):
        samples = []
        for r in range(repetitions + warmup):
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.record()
            fn()
            en.record()
            en.synchronize()
            if r >= warmup:
                samples.append(st.elapsed_time(en))
        samples.sort()
        p90 = samples[min(len(samples) - 1, int(round(0.9 * (len(samples) - 1))))]
        return {"median": statistics.median(samples), "p90": p90, "n": len(samples),
                "flag": "no-variance" if len(samples) == 1 else None}

    geom = weight.geom
    base = timeit(lambda: me_linear(x, weight, None, [], geom=geom))  # noqa: E731
    delta = timeit(lambda: me_linear(x, None, table, segments, geom=geom)) if segments else \
        {"median": 0.0, "p90": 0.0, "n": 0, "flag": None}
    total = timeit(lambda: me_linear(x, weight, table, segments, geom=geom))
    return {"base_gemm_ms": base, "delta_stage_ms": delta, "total_ms": total}
