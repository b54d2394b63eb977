"""Per-linear parity checker for the Mistral-shaped serving engine (TEST INFRASTRUCTURE ONLY).

Used by tests/test_gpu_mistral_full.py and, outside the timed region, by bench.py's parity
block.  Hooked into `MistralMultiExpert.step(trace=...)`, it reads back the exact bf16 input
rows and output rows of every fused linear launch of the sampled layers and compares them
with the f64 restatement of Eq. 4 on those identical inputs:

    y_ref[r] = x[r] . W  +  delta_matvec(x[r], expert(r))  (+ residual[r])

where W is the engine's bf16 base weight (read back through the debug relayout) and
delta_matvec is oracle/mesw.delta_matvec_batch (s_j * sum_{i not in S} x_i
q_ij + sum_{i in S} x_i half(R_i)_j, f64, from the artifact's packed codes -- compress.py:
115-121, quant.py:216-236).  The metric is max |y - y_ref| / max |y_ref| over the rows that
hold requests (north_star: <= 1e-2), plus argmax agreement of the final logits (first
maximum, toylm.py:247) against the f64 logits.
"""

from __future__ import annotations

import numpy as np

from . import mesw as om

PROJ_ORDER = ("q", "k", "v", "o", "gate", "up", "down")
KIND_PROJ = {"qkv": ("q", "k", "v"), "o": ("o",), "gu": ("gate", "up"), "down": ("down",), "head": ()}


class LinearParity:
    """trace(when, kind, layer, r0, r1, bufs) hook for MistralMultiExpert.step.

    experts: {expert_id: list of oracle layers (7 per decoder layer, artifact order)}.
    layers: decoder layers to check (others run unchecked); head: check lm_head too."""

    def __init__(self, eng, experts: dict, layers=(0,), head: bool = True):
        self.eng = eng
        self.experts = experts
        self.layers = set(layers)
        self.head = head
        self.results = []  # (kind, layer, group r0, max_rel_err, rows)
        self.argmax = []   # per checked head group: (agree, rows)
        self._pre = {}
        self._w = {}

    # ---------------------------------------------------------------- readback helpers
    def _weight(self, kind, layer):
        key = (kind, layer)
        if key not in self._w:
            eng = self.eng
            if kind == "head":
                dw = eng.head
            else:
                lw = eng.layers[layer]
                dw = {"qkv": lw.qkv, "o": lw.o, "gu": lw.gateup, "down": lw.down}[kind]
            self._w = {key: [dw.dense(b).float().cpu().numpy().astype(np.float64)
                             for b in range(len(dw.geom.block_n))]}
        return self._w[key]

    def _input(self, kind, r0, r1, bufs):
        from paper_2406_09041_b200.device import unpack_x
        eng = self.eng
        name = {"qkv": "xn", "gu": "xn", "head": "xn", "o": "attn", "down": "act"}[kind]
        m = {"qkv": eng.g_qkv.m, "gu": eng.g_gu.m, "head": eng.g_head.m, "o": eng.g_o.m, "down": eng.g_down.m}[kind]
        return unpack_x(bufs[name], r1 - r0, m).float().cpu().numpy().astype(np.float64)

    def _output(self, kind, r0, r1):
        eng = self.eng
        t = {"qkv": eng.qkv, "gu": eng.gu, "o": eng.h, "down": eng.h, "head": eng.logits}[kind]
        return t[r0:r1].float().cpu().numpy().astype(np.float64)

    def _geom(self, kind):
        eng = self.eng
        return {"qkv": eng.g_qkv, "gu": eng.g_gu, "o": eng.g_o, "down": eng.g_down, "head": eng.g_head}[kind]

    # ---------------------------------------------------------------- hook
    def __call__(self, when, kind, layer, r0, r1, bufs):
        if kind == "head" and not self.head:
            return
        if kind != "head" and layer not in self.layers:
            return
        import torch
        torch.cuda.synchronize()
        if when == "pre":
            res = self._output(kind, r0, r1) if kind in ("o", "down") else None
            self._pre[(kind, layer, r0)] = (self._input(kind, r0, r1, bufs), res)
            return
        x, res = self._pre.pop((kind, layer, r0))
        y = self._output(kind, r0, r1)
        geom = self._geom(kind)
        W = self._weight(kind, layer)
        eng = self.eng
        rows = np.arange(r0, r1)
        real = eng.rows[rows] >= 0  # rows that hold requests
        slot_of = np.full(r1 - r0, -1)
        for b, e, sl in eng.segments:
            lo, hi = max(b, r0), min(e, r1)
            if lo < hi:
                slot_of[lo - r0:hi - r0] = sl
        id_of_slot = {sl: eid for eid, (sl, _) in eng.experts.items()}
        ref = np.zeros((r1 - r0, geom.n_pad))
        for bi, (cb, nb) in enumerate(zip(geom.col_base, geom.block_n)):
            ref[:, cb:cb + nb] = x @ W[bi]
            if kind == "head":
                continue
            proj = KIND_PROJ[kind][bi]
            for sl in sorted(set(slot_of[real].tolist()) - {-1}):
                sel = np.flatnonzero((slot_of == sl) & real)
                blk = self.experts[id_of_slot[sl]][7 * layer + PROJ_ORDER.index(proj)]
                ref[sel, cb:cb + nb] += om.delta_matvec_batch(x[sel], blk)
        if res is not None:
            ref += res[:, :geom.n_pad] if res.shape[1] >= geom.n_pad else np.pad(res, ((0, 0), (0, geom.n_pad - res.shape[1])))
        cols = np.concatenate([np.arange(cb, cb + nb) for cb, nb in zip(geom.col_base, geom.block_n)])
        yr, rr = y[real][:, cols], ref[real][:, cols]
        err = float(np.max(np.abs(yr - rr)) / max(np.max(np.abs(rr)), 1e-30))
        self.results.append((kind, layer, r0, err, int(real.sum())))
        if kind == "head":
            V = eng.shape.vocab
            got = np.argmax(y[real][:, :V], axis=-1)  # first maximum, as mesw_argmax / np.argmax
            want = np.argmax(ref[real][:, :V], axis=-1)
            self.argmax.append((float(np.mean(got == want)), int(real.sum())))

    # ---------------------------------------------------------------- summary
    def max_rel_err(self) -> float:
        return max((r[3] for r in self.results), default=float("nan"))

    def argmax_agree(self) -> float:
        n = sum(c for _, c in self.argmax)
        return sum(a * c for a, c in self.argmax) / n if n else float("nan")

    def summary(self) -> dict:
        return {"max_rel_err": self.max_rel_err(), "argmax_agree": self.argmax_agree(),
                "linears_checked": len(self.results),
                "per_linear": [{"kind": k, "layer": l, "rows_from": r0, "max_rel_err": e, "rows": n}
                               for k, l, r0, e, n in self.results]}
