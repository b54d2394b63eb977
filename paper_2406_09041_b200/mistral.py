"""Mistral-7B-shaped multi-expert decode engine (BASELINE configs 2 and 3).

One shared bf16 base model; every request carries an expert id whose compressed
delta (2-bit codes + fp16 salient rows) is applied inside the four fused linears
of every decoder layer (q|k|v, o, gate|up, down -- 7 compressed projections, the
224 decoder linears the paper's 2.13 GB Mistral delta covers).
Embedding and lm_head are base-only.

Requests are kept grouped by expert for the whole batch lifetime, so each fused
linear sees fixed segments; the per-step launch sequence (all CUDA kernels from
libmesw.so) is captured once in a CUDA graph and replayed.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import (DeviceDelta, DeviceWeight, ExpertTable, LinearGeometry, LinearPlan, _stream,
                     Workspace, canonical_numel, canonical_rows, corr_table, cta_candidates, tune_num_ctas)
from .synth import MistralShape

# rope + KV-cache append run inside the attention launch (mesw_attention_decode_rope)
_FUSED_ROPE = os.environ.get("MESW_ROPE_SPLIT") is None
# SwiGLU in the gate|up launch's epilogue (mesw_linear_args.swiglu_I) saves one launch per
# layer but lengthens the gate|up tail (the second finisher of each gate/up block pair reads
# both halves back from L2): measured 6.13 vs 6.09 ms per C2 step, so it is opt-in
# (MESW_SWIGLU_FUSED=1) and the separate mesw_swiglu launch stays the default.
_FUSED_SWIGLU = os.environ.get("MESW_SWIGLU_FUSED") is not None

PROJ_ORDER = ("q", "k", "v", "o", "gate", "up", "down")
MAX_EXPERT_SLOTS = 128  # resident experts per engine (C5: 64 on one GPU)


@dataclass
class LayerWeights:
    attn_norm: torch.Tensor
    qkv: DeviceWeight
    o: DeviceWeight
    mlp_norm: torch.Tensor
    gateup: DeviceWeight
    down: DeviceWeight


def _launch_groups(B: int, segs: list) -> list:
    """Launch groups of the engine rows (device.launch_groups: row and TMEM budgets)."""
    from .device import launch_groups
    return launch_groups(B, segs)


class CacheWindowError(ValueError):
    """A decode step would write past a request's KV-cache window (ctx_max)."""


class MistralMultiExpert:
    """Base model + resident experts + decode buffers for up to `max_batch` requests."""

    def __init__(self, shape: MistralShape = MistralShape(), max_batch: int = 64, ctx_max: int = 256,
                 device="cuda", n_layers: int | None = None, offset_codes: bool = True, tune: bool = True):
        self.shape = shape
        self.tune = tune  # time candidate launch widths per linear kind once per batch layout
        self.offset_codes = offset_codes  # 2-bit codes in offset form + glue-written bias tables
        self.n_layers = shape.n_layers if n_layers is None else n_layers
        self.device = torch.device(device)
        self.max_batch = max_batch
        self.ctx_max = ctx_max
        s = shape
        self.kv_dim = s.n_kv_heads * s.head_dim
        self.g_qkv = LinearGeometry(s.hidden, (s.n_heads * s.head_dim, self.kv_dim, self.kv_dim))
        self.g_o = LinearGeometry(s.n_heads * s.head_dim, (s.hidden,))
        self.g_gu = LinearGeometry(s.hidden, (s.intermediate, s.intermediate))
        self.g_down = LinearGeometry(s.intermediate, (s.hidden,))
        self.g_head = LinearGeometry(s.hidden, (s.vocab,))
        self.layers: list[LayerWeights] = []
        # fixed capacity: launch plans bind the tables' device pointers (a table never regrows here)
        self.tables = [[ExpertTable(self.device, capacity=MAX_EXPERT_SLOTS) for _ in range(4)]
                       for _ in range(self.n_layers)]
        self.experts: dict = {}
        self.embedding = None
        self.final_norm = None
        self.head = None
        self._alloc_buffers()
        self.graph = None
        self._plans = None
        # benchmark steady state only: a request reaching ctx_max wraps back to position 128
        # (its cache rows are overwritten).  Serving (False) raises CacheWindowError instead.
        self.wrap_positions = False
        self._pos_max = 0
        self.registry = None
        self._pinned = []

    # ------------------------------------------------------------------ weights
    def _alloc_buffers(self):
        s, B, dev = self.shape, self.max_batch, self.device
        bf = torch.bfloat16
        self.ids = torch.zeros(B, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(B, dtype=torch.int32, device=dev)
        self.len = torch.ones(B, dtype=torch.int32, device=dev)
        self.h = torch.zeros((B, s.hidden), dtype=bf, device=dev)
        # (the fused linears' inputs live in per-launch-group canonical buffers: _build_plans)
        self.qkv = torch.zeros((B, self.g_qkv.n_pad), dtype=bf, device=dev)
        self.gu = torch.zeros((B, self.g_gu.n_pad), dtype=bf, device=dev)
        # f32 logits: greedy argmax over bf16-rounded logits would tie / misorder near-equal
        # candidates (a 32000-way argmax; the f32 epilogue value is what the reference compares)
        self.logits = torch.zeros((B, self.g_head.n_pad), dtype=torch.float32, device=dev)
        kv_shape = (self.n_layers, B, self.ctx_max, s.n_kv_heads, s.head_dim)
        self.kcache = torch.zeros(kv_shape, dtype=bf, device=dev)
        self.attn_ws = torch.empty(int(_lib.lib().mesw_attention_workspace_bytes(B, s.n_heads, self.ctx_max)),
                                   dtype=torch.uint8, device=dev)
        self.vcache = torch.zeros(kv_shape, dtype=bf, device=dev)

    def load_base(self, embedding, final_norm, head_w, layers: list) -> None:
        """Install base weights.  `layers[l]` = dict(attn_norm, q, k, v, o, mlp_norm, gate, up, down)
        with projection matrices in reference orientation [in, out] (bf16/f32 tensors)."""
        dev = self.device
        self.embedding = torch.as_tensor(embedding).to(dev, torch.bfloat16).contiguous()
        self.final_norm = torch.as_tensor(final_norm).to(dev, torch.bfloat16).contiguous()
        self.head = DeviceWeight.empty(self.g_head, dev)
        self.head.load_block(0, torch.as_tensor(head_w).to(dev))
        self.layers = []
        for lw in layers:
            qkv = DeviceWeight.empty(self.g_qkv, dev)
            for b, name in enumerate(("q", "k", "v")):
                qkv.load_block(b, torch.as_tensor(lw[name]).to(dev))
            o = DeviceWeight.empty(self.g_o, dev)
            o.load_block(0, torch.as_tensor(lw["o"]).to(dev))
            gu = DeviceWeight.empty(self.g_gu, dev)
            gu.load_block(0, torch.as_tensor(lw["gate"]).to(dev))
            gu.load_block(1, torch.as_tensor(lw["up"]).to(dev))
            down = DeviceWeight.empty(self.g_down, dev)
            down.load_block(0, torch.as_tensor(lw["down"]).to(dev))
            self.layers.append(LayerWeights(
                attn_norm=torch.as_tensor(lw["attn_norm"]).to(dev, torch.bfloat16).contiguous(), qkv=qkv, o=o,
                mlp_norm=torch.as_tensor(lw["mlp_norm"]).to(dev, torch.bfloat16).contiguous(), gateup=gu, down=down))
        self._plans = None

    def load_synthetic_base(self, seed: int = 0, std: float = 0.02) -> None:
        """Random-init base weights of the Mistral architecture (no checkpoints offline),
        generated on the device block by block."""
        s, dev = self.shape, self.device
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def rnd(*shape):
            return (torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * std).to(torch.bfloat16)

        self.embedding = rnd(s.vocab, s.hidden)
        self.final_norm = torch.ones(s.hidden, dtype=torch.bfloat16, device=dev)
        self.head = DeviceWeight.empty(self.g_head, dev)
        self.head.load_block(0, rnd(s.hidden, s.vocab))
        self.layers = []
        for _ in range(self.n_layers):
            qkv = DeviceWeight.empty(self.g_qkv, dev)
            for b, nb in enumerate(self.g_qkv.block_n):
                qkv.load_block(b, rnd(s.hidden, nb))
            o = DeviceWeight.empty(self.g_o, dev)
            o.load_block(0, rnd(self.g_o.m, s.hidden))
            gu = DeviceWeight.empty(self.g_gu, dev)
            gu.load_block(0, rnd(s.hidden, s.intermediate))
            gu.load_block(1, rnd(s.hidden, s.intermediate))
            down = DeviceWeight.empty(self.g_down, dev)
            down.load_block(0, rnd(s.intermediate, s.hidden))
            ones = torch.ones(s.hidden, dtype=torch.bfloat16, device=dev)
            self.layers.append(LayerWeights(attn_norm=ones, qkv=qkv, o=o, mlp_norm=ones.clone(), gateup=gu,
                                            down=down))
        torch.cuda.synchronize(dev)
        self._plans = None

    def base_bytes(self) -> int:
        n = sum(t.numel() * t.element_size() for lw in self.layers for t in
                (lw.qkv.frag, lw.o.frag, lw.gateup.frag, lw.down.frag))
        return n + self.head.frag.numel() * 2

    # ------------------------------------------------------------------ experts
    def _fused_blocks(self, artifact) -> list:
        """Per layer: the blocks of the 4 fused linears (q|k|v, o, gate|up, down) with their geometry."""
        layers = artifact.layers if hasattr(artifact, "layers") else list(artifact)
        if len(layers) != 7 * self.n_layers:
            raise ValueError(f"expert artifact has {len(layers)} blocks, expected {7 * self.n_layers}")
        out = []
        for l in range(self.n_layers):
            blk = dict(zip(PROJ_ORDER, layers[7 * l:7 * l + 7]))
            out.append((([blk["q"], blk["k"], blk["v"]], self.g_qkv), ([blk["o"]], self.g_o),
                        ([blk["gate"], blk["up"]], self.g_gu), ([blk["down"]], self.g_down)))
        return out

    def load_deltas(self, artifact, stream=None) -> list:
        """Upload + repack an expert (pinned staging, async copies and K1 on `stream`):
        [layer][linear kind] DeviceDelta."""
        staging: list = []
        deltas = [[DeviceDelta.from_blocks(b, g, self.device, stream=stream, staging=staging) for b, g in kinds]
                  for kinds in self._fused_blocks(artifact)]
        (stream if stream is not None else torch.cuda.current_stream(self.device)).synchronize()
        return deltas

    def expert_device_bytes(self, artifact) -> int:
        """HBM bytes an expert will occupy in this engine (the registry budget unit)."""
        return sum(DeviceDelta.device_nbytes(b, g) for kinds in self._fused_blocks(artifact) for b, g in kinds)

    def _install(self, expert_id, deltas) -> int:
        used = {sl for sl, _ in self.experts.values()}
        slot = next(i for i in range(len(used) + 1) if i not in used)  # lowest free slot
        if slot >= MAX_EXPERT_SLOTS:
            raise ValueError(f"more than {MAX_EXPERT_SLOTS} resident experts")
        nbytes = 0
        for l, per in enumerate(deltas):
            for t, d in zip(self.tables[l], per):
                t.set(slot, d)
                nbytes += d.nbytes
        self.experts[expert_id] = (slot, nbytes)
        return slot

    def _uninstall(self, expert_id) -> None:
        slot, _ = self.experts.pop(expert_id)
        for per in self.tables:
            for t in per:
                t.set(slot, None)

    def add_expert(self, expert_id, artifact) -> int:
        """Make an expert resident: its artifact holds 7 blocks per layer (q,k,v,o,gate,up,down)."""
        slot = self._install(expert_id, self.load_deltas(artifact))
        self._plans = None
        self.graph = None
        return slot

    def expert_bytes(self) -> int:
        return sum(nb for _, nb in self.experts.values())

    # ------------------------------------------------------------------ registry (on-demand experts)
    def make_registry(self, budget_bytes: int, base_digest: str):
        """An `ExpertRegistry` that owns this engine's expert residency:
        `set_batch` acquires (loads on demand, pins) the batch's experts and releases the
        previous batch's with a fence on the decode stream; eviction (strict LRU over
        unpinned experts) waits for that fence, then frees the expert's table slot.  The
        budget counts HBM bytes (`expert_device_bytes`); loads run on a copy stream from
        pinned host buffers."""
        from .registry import ExpertRegistry, GpuHandle

        eng = self

        class EngineExpert(GpuHandle):
            def __init__(self, deltas):
                self.deltas = deltas
                self.device_bytes = sum(d.nbytes for per in deltas for d in per)

        def load(expert_id, artifact):
            h = EngineExpert(eng.load_deltas(artifact, stream=eng._copy_stream()))
            eng._install(expert_id, h.deltas)
            return h

        def unload(expert_id, handle):
            if expert_id in eng.experts:
                eng._uninstall(expert_id)

        self.registry = ExpertRegistry(budget_bytes, base_digest, loader=load, unloader=unload,
                                       size_fn=self.expert_device_bytes)
        self._pinned = []
        return self.registry

    def _copy_stream(self):
        if getattr(self, "_cstream", None) is None:
            self._cstream = torch.cuda.Stream(device=self.device)
        return self._cstream

    # ------------------------------------------------------------------ batch
    def set_batch(self, expert_ids: list, prompt_lens: list | None = None) -> np.ndarray:
        """Fix the request batch.  Requests are regrouped by expert; every expert group starts
        on a 16-row tcgen05 window, or on an 8-row half window when it holds <= 8 requests
        (device.segment_align: two small experts share a window); padding rows are inert.  Returns `rows`: rows[r] = caller's request index at engine row r
        (-1 for padding).  Positions start at prompt_lens (cache rows below are assumed
        filled)."""
        n = len(expert_ids)
        if n < 1:
            raise ValueError("empty batch")
        reg = getattr(self, "registry", None)
        if reg is not None:  # on-demand residency: pin this batch's experts, unpin the last batch's
            want = list(dict.fromkeys(e for e in expert_ids if e is not None))
            stream = torch.cuda.current_stream(self.device)
            for e in self._pinned:
                reg.release(e, stream)
            self._pinned = []
            try:
                for e in want:
                    reg.acquire(e)
                    self._pinned.append(e)
            except BaseException:
                for e in self._pinned:
                    reg.release(e, stream)
                self._pinned = []
                raise
        slots = []
        for e in expert_ids:
            if e is None:
                slots.append(-1)
            elif e not in self.experts:
                from .errors import UnknownExpertError
                raise UnknownExpertError(f"unknown expert {e!r}")
            else:
                slots.append(self.experts[e][0])
        slots = np.asarray(slots)
        rows, segs = [], []
        from .device import segment_align
        for sl in sorted(set(slots.tolist()) - {-1}):
            members = np.flatnonzero(slots == sl).tolist()
            while len(rows) % segment_align(len(members)):  # <= 8 requests: half a 16-row window
                rows.append(-1)
            segs.append((len(rows), len(rows) + len(members), int(sl)))
            rows.extend(members)
        rows.extend(np.flatnonzero(slots == -1).tolist())  # base-only requests
        B = len(rows)
        if B > self.max_batch:
            raise ValueError(f"padded batch of {B} rows exceeds max_batch={self.max_batch}")
        rows = np.asarray(rows)
        pl_req = np.zeros(n, np.int64) if prompt_lens is None else np.asarray(prompt_lens, np.int64)
        if (pl_req >= self.ctx_max).any():
            raise ValueError("prompt longer than the cache window")
        pl = np.where(rows >= 0, pl_req[np.maximum(rows, 0)], 0)
        groups = _launch_groups(B, segs)
        if getattr(self, "B", None) != B or getattr(self, "segments", None) != segs:
            self._plans = None  # launch geometry changed: rebuild plans / re-capture
            self.graph = None
        self.groups = groups
        self.B = B
        self.n_requests = n
        self.rows = rows
        self.order = rows
        self.segments = segs
        self.pos[:B] = torch.as_tensor(pl, dtype=torch.int32)
        self.len[:B] = torch.as_tensor(pl + 1, dtype=torch.int32)
        self._pos_max = int(pl.max())
        return rows

    def fill_random_kv(self, prompt_len: int, seed: int = 1) -> None:
        """Synthetic prompt state: random K/V for positions < prompt_len (bench only)."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        for t in (self.kcache, self.vcache):
            for l in range(t.shape[0]):  # per layer: bounded temporaries (many-expert engines)
                view = t[l, :, :prompt_len]
                view.copy_((torch.randn(view.shape, generator=g, device=self.device) * 0.5).to(torch.bfloat16))

    # ------------------------------------------------------------------ step
    def _build_plans(self):
        """Per launch group (rows [r0, r1), <= MAX_ROWS padded rows, segments rebased): its
        canonical input buffers and the fused-linear plans of every layer + lm_head."""
        s = self.shape
        gplans = []
        for (r0, r1, segs) in self.groups:
            rows = r1 - r0
            bufs = {
                "xn": torch.zeros(canonical_numel(rows, s.hidden), dtype=torch.bfloat16, device=self.device),
                "attn": torch.zeros(canonical_numel(rows, self.g_o.m), dtype=torch.bfloat16, device=self.device),
                "act": torch.zeros(canonical_numel(rows, self.g_down.m), dtype=torch.bfloat16, device=self.device),
            }
            # offset-code bias tables written by the glue next to each canonical input (mesw.h x_corr)
            for k, m in (("xn", s.hidden), ("attn", self.g_o.m), ("act", self.g_down.m)):
                bufs[k + "_corr"] = corr_table(rows, m, self.device) if self.offset_codes else None
            h, qkv, gu = self.h[r0:r1], self.qkv[r0:r1], self.gu[r0:r1]
            # per linear kind: (input, weight of layer l, table index, output, residual?)
            kinds = (("qkv", "xn", lambda lw: lw.qkv, 0, qkv, False), ("o", "attn", lambda lw: lw.o, 1, h, True),
                     ("gu", "xn", lambda lw: lw.gateup, 2, gu, False), ("down", "act", lambda lw: lw.down, 3, h, True))
            ctas = {}
            for name, xin, wsel, ti, out, res in kinds:
                ctas[name] = self._tuned_ctas(name, rows, segs, bufs[xin], bufs[xin + "_corr"], wsel(self.layers[0]),
                                              self.tables[0][ti] if segs else None, out, res)
            layers = []
            for l, lw in enumerate(self.layers):
                tabs = self.tables[l]
                layers.append(tuple(
                    LinearPlan(bufs[xin], rows, wsel(lw), tabs[ti] if segs else None, segs, out,
                               residual=out if res else None, x_corr=bufs[xin + "_corr"], num_ctas=ctas[name],
                               swiglu=(s.intermediate, bufs["act"], bufs["act_corr"])
                               if (name == "gu" and _FUSED_SWIGLU) else None)
                    for name, xin, wsel, ti, out, res in kinds))
            head = LinearPlan(bufs["xn"], rows, self.head, None, [], self.logits[r0:r1],
                              num_ctas=self._tuned_ctas("head", rows, [], bufs["xn"], None, self.head, None,
                                                        self.logits[r0:r1], False))
            gplans.append((r0, r1, bufs, layers, head))
        self._plans = gplans

    def _tuned_ctas(self, name, rows, segs, xc, corr, weight, table, out, res) -> int:
        """Launch width of one linear kind for this batch layout, timed on scratch outputs
        (device.tune_num_ctas; cached per shape key).  0 = one CTA per SM."""
        if not self.tune:
            return 0
        key = ("mistral", name, self.shape, rows, tuple((b, e) for b, e, _ in segs),
               table.code_bits if table is not None else 0, corr is not None)
        scratch = torch.empty_like(out)

        def make(c):
            return LinearPlan(xc, rows, weight, table, segs, scratch, residual=scratch if res else None,
                              x_corr=corr, num_ctas=c)
        sms = Workspace.get(self.device).sms
        return tune_num_ctas(key, make, cta_candidates(weight.geom, sms))

    def step(self, stream=None, trace=None) -> None:
        """One decode step for the whole batch: ids (engine order) -> next ids in self.ids.
        Batches wider than one fused launch (> MAX_ROWS padded rows, e.g. many experts)
        run as several launch groups; each re-streams the base weights.

        trace (parity checks, eager only): called as trace(when, kind, layer, r0, r1, bufs)
        with when in ("pre", "post") around every fused linear launch (kind in "qkv", "o",
        "gu", "down", "head"), so a checker can read the exact bf16 inputs and outputs."""
        if self._plans is None:
            self._build_plans()
        L = _lib.lib()
        st = _stream(stream)
        s, B = self.shape, self.B
        chk = _lib.check
        H = s.hidden
        eps = C.c_float(s.rms_eps)
        bf = 2  # bytes per bf16

        def rows_ptr(t, r0):
            return t.data_ptr() + r0 * t.stride(0) * bf

        def corr(bufs, k):  # (pointer, leading dimension) of a bias table, or none
            c = bufs[k + "_corr"]
            return (c.data_ptr(), c.stride(0)) if c is not None else (None, 0)

        chk(L.mesw_embed(self.ids.data_ptr(), B, self.embedding.data_ptr(), H, self.h.data_ptr(),
                         self.h.stride(0), st))
        for l, lw in enumerate(self.layers):
            for (r0, r1, bufs, layers, _) in self._plans:
                chk(L.mesw_rmsnorm(rows_ptr(self.h, r0), self.h.stride(0), lw.attn_norm.data_ptr(), r1 - r0, H, eps,
                                   bufs["xn"].data_ptr(), 0, canonical_rows(r1 - r0), *corr(bufs, "xn"), st))
                if trace:
                    trace("pre", "qkv", l, r0, r1, bufs)
                layers[l][0](stream)
                if trace:
                    trace("post", "qkv", l, r0, r1, bufs)
            kc, vc = self.kcache[l], self.vcache[l]
            if not _FUSED_ROPE:  # two-call form (A/B switch MESW_ROPE_SPLIT=1)
                chk(L.mesw_rope_append(self.qkv.data_ptr(), self.qkv.stride(0), self.pos.data_ptr(), B, s.n_heads,
                                       s.n_kv_heads, s.head_dim, C.c_float(s.rope_theta), kc.data_ptr(),
                                       vc.data_ptr(), self.ctx_max, st))
            for (r0, r1, bufs, layers, _) in self._plans:
                if _FUSED_ROPE:  # rope + KV append folded into the attention launch (len = pos + 1)
                    chk(L.mesw_attention_decode_rope(
                        rows_ptr(self.qkv, r0), self.qkv.stride(0), rows_ptr(kc, r0), rows_ptr(vc, r0),
                        self.len.data_ptr() + 4 * r0, r1 - r0, s.n_heads, s.n_kv_heads, s.head_dim,
                        C.c_float(s.rope_theta), self.ctx_max, bufs["attn"].data_ptr(), 0, canonical_rows(r1 - r0),
                        self.attn_ws.data_ptr(), self.attn_ws.numel(), *corr(bufs, "attn"), st))
                else:
                    chk(L.mesw_attention_decode(rows_ptr(self.qkv, r0), self.qkv.stride(0), rows_ptr(kc, r0),
                                                rows_ptr(vc, r0), self.len.data_ptr() + 4 * r0, r1 - r0, s.n_heads,
                                                s.n_kv_heads, s.head_dim, self.ctx_max, bufs["attn"].data_ptr(), 0,
                                                canonical_rows(r1 - r0), self.attn_ws.data_ptr(),
                                                self.attn_ws.numel(), *corr(bufs, "attn"), st))
                if trace:
                    trace("pre", "o", l, r0, r1, bufs)
                layers[l][1](stream)
                if trace:
                    trace("post", "o", l, r0, r1, bufs)
            for (r0, r1, bufs, layers, _) in self._plans:
                chk(L.mesw_rmsnorm(rows_ptr(self.h, r0), self.h.stride(0), lw.mlp_norm.data_ptr(), r1 - r0, H, eps,
                                   bufs["xn"].data_ptr(), 0, canonical_rows(r1 - r0), *corr(bufs, "xn"), st))
                if trace:
                    trace("pre", "gu", l, r0, r1, bufs)
                layers[l][2](stream)
                if trace:
                    trace("post", "gu", l, r0, r1, bufs)
            for (r0, r1, bufs, layers, _) in self._plans:
                if not _FUSED_SWIGLU:  # (fused: the gate|up launch wrote act and its bias table)
                    chk(L.mesw_swiglu(rows_ptr(self.gu, r0), self.gu.stride(0), r1 - r0, s.intermediate,
                                      bufs["act"].data_ptr(), 0, canonical_rows(r1 - r0), *corr(bufs, "act"), st))
                if trace:
                    trace("pre", "down", l, r0, r1, bufs)
                layers[l][3](stream)
                if trace:
                    trace("post", "down", l, r0, r1, bufs)
        for (r0, r1, bufs, _, head) in self._plans:
            chk(L.mesw_rmsnorm(rows_ptr(self.h, r0), self.h.stride(0), self.final_norm.data_ptr(), r1 - r0, H, eps,
                               bufs["xn"].data_ptr(), 0, canonical_rows(r1 - r0), None, 0, st))
            if trace:
                trace("pre", "head", -1, r0, r1, bufs)
            head(stream)
            if trace:
                trace("post", "head", -1, r0, r1, bufs)
        chk(L.mesw_argmax(self.logits.data_ptr(), 0, B, s.vocab, self.logits.stride(0), self.ids.data_ptr(), st))
        wrap_to = min(self.ctx_max - 1, 128) if self.wrap_positions else -1
        chk(L.mesw_advance_positions(self.pos.data_ptr(), self.len.data_ptr(), B, self.ctx_max, wrap_to, st))

    def launches_per_step(self) -> int:
        g = len(self.groups)
        per_layer = g * 9 + (0 if _FUSED_ROPE else 1)  # attention is 2 kernels (rope folded in)
        return 1 + per_layer * self.n_layers + g * 2 + 2

    def capture(self) -> None:
        """Capture one decode step in a CUDA graph (replayed by `replay`).  The warm-up step
        (kernel attributes, launch-width tuning) runs eagerly, so the decode state it
        advances -- ids, positions, lengths -- is restored afterwards; the KV row it wrote
        is rewritten by the next real step at the same position."""
        B = self.B
        saved = (self.ids[:B].clone(), self.pos[:B].clone(), self.len[:B].clone())
        self.step()  # warm: configures kernel attributes outside capture
        self.ids[:B].copy_(saved[0])
        self.pos[:B].copy_(saved[1])
        self.len[:B].copy_(saved[2])
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            g.capture_begin()
            self.step(stream=s)
            g.capture_end()
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.graph = g

    def _advance_host(self) -> None:
        """Host-side cache-window check before a step (positions advance on the device)."""
        if not self.wrap_positions:
            if self._pos_max >= self.ctx_max:
                raise CacheWindowError(f"a request reached the cache window (ctx_max={self.ctx_max}); "
                                       "finish or re-batch it before the next step")
            self._pos_max += 1

    def replay(self) -> None:
        if self.graph is None:
            self.capture()
        self._advance_host()
        self.graph.replay()

    def bytes_per_step(self) -> dict:
        """Algorithmic HBM bytes of one decode step."""
        s, B = self.shape, self.B
        from .synth import linear_bytes
        n_exp = len(self.segments)
        lin = 0
        delta = 0
        base = 0
        for g in (self.g_qkv, self.g_o, self.g_gu, self.g_down):
            lin += linear_bytes(g.m, g.n, n_exp, B)
            delta += linear_bytes(g.m, g.n, n_exp, B, base=False) - 2 * B * (g.m + g.n)
            base += linear_bytes(g.m, g.n, 0, B)
        lin *= self.n_layers
        delta *= self.n_layers
        base *= self.n_layers
        head = linear_bytes(s.hidden, s.vocab, 0, B)
        ctx = int(self.len[:B].float().mean().item())
        kv = 2 * B * ctx * s.n_kv_heads * s.head_dim * 2 * self.n_layers
        return {"linears": lin, "delta": delta, "base_linears": base, "head": head, "kv": kv,
                "total": lin + head + kv}

    # ------------------------------------------------------------------ public API
    def decode(self, host_ids: torch.Tensor, out_host: torch.Tensor | None = None) -> torch.Tensor:
        """End-to-end step through the public API: host token ids (engine order, int32,
        pinned) -> device, one graph-replayed decode step, next ids -> host."""
        B = self.B
        self.ids[:B].copy_(host_ids[:B], non_blocking=True)
        self.replay()
        if out_host is None:
            out_host = torch.empty(B, dtype=torch.int32, pin_memory=True)
        out_host.copy_(self.ids[:B], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return out_host
