"""f3: step-size distillation on the GPU -- drop-in for compress.distill_step_sizes
(compress.py:331-378).

Only the step vectors move: every batch re-quantizes each layer's raw delta at the
current steps (QuantizedLayerState.reconstruct, toylm.py:379-384), runs the toy model
forward and the exact reverse pass (toylm.py:394-447), contracts each layer's upstream
gradient with the straight-through quantizer rule (quant.py:142-169) and applies the
AdamW-rule update with f64 moments (compress.py:276-302) and the positive clamp.

Per layer the quantizer work runs in sm_100a kernels (include/mesw.h f3:
mesw_ste_reconstruct fused with `w + d`, mesw_ste_step_grad, mesw_adam_step,
mesw_quantize_pack for the final _repack), each bit-exact with the reference's numpy
for the same inputs.  The model's GEMMs are plain f32 cuBLAS calls through torch (TF32
off); they round differently from OpenBLAS, so end-to-end results match the reference
within f32 tolerance (tests/test_gpu_distill.py), not bit-for-bit.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .compress import CompressedDelta, PackedCodes
from .errors import DistillDivergenceError
from .infer import _positional_bias

__all__ = ["DistillConfig", "DistillResult", "STEP_FLOOR", "distill_step_sizes", "backward_step_sizes"]

STEP_FLOOR = 1e-8  # compress.py:305


@dataclass(frozen=True)
class DistillConfig:
    """compress.py:66-70."""
    epochs: int = 1
    lr: float = 1e-5
    batch_size: int = 4


@dataclass
class DistillResult:
    """compress.py:308-313."""
    layers: list
    initial_loss: float
    final_loss: float
    batch_losses: list


def _stream(torch, dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


class _LayerState:
    """toylm.QuantizedLayerState (toylm.py:357-391) with device buffers."""

    def __init__(self, torch, delta, art, dev):
        self.torch, self.dev = torch, dev
        self.delta = delta  # f32 [m, n] on the device
        m, n = delta.shape
        self.m, self.n, self.bits = m, n, int(art.bits)
        idx = np.asarray(art.salient.indices, np.int64)
        self.k = idx.size
        slot = np.full(m, -1, np.int32)
        slot[idx] = np.arange(idx.size, dtype=np.int32)
        self.row_slot = torch.from_numpy(slot).to(dev) if idx.size else None
        self.sal_rows = (torch.from_numpy(np.asarray(art.salient_rows, np.float16).astype(np.float32)).to(dev)
                         if idx.size else None)
        self.mask = torch.from_numpy((slot >= 0).astype(np.uint8)).to(dev)
        self.steps = torch.from_numpy(np.asarray(art.steps, np.float32).copy()).to(dev)

    def effective(self, base_w, out):
        """out = base_w + reconstruct() (toylm.py:422-424)."""
        _lib.check(_lib.lib().mesw_ste_reconstruct(
            self.delta.data_ptr(), self.m, self.n, self.steps.data_ptr(), self.bits,
            self.row_slot.data_ptr() if self.row_slot is not None else None,
            self.sal_rows.data_ptr() if self.sal_rows is not None else None,
            base_w.data_ptr(), out.data_ptr(), _stream(self.torch, self.dev)))
        return out

    def step_gradient(self, upstream):
        up = upstream.contiguous()
        g = self.torch.empty(self.n, dtype=self.torch.float32, device=self.dev)
        _lib.check(_lib.lib().mesw_ste_step_grad(
            self.delta.data_ptr(), self.m, self.n, self.steps.data_ptr(), self.bits,
            self.row_slot.data_ptr() if self.row_slot is not None else None,
            up.data_ptr(), g.data_ptr(), _stream(self.torch, self.dev)))
        return g


class _Adam:
    """compress._Adam (compress.py:276-302) over device step vectors."""

    def __init__(self, torch, states, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.torch, self.lr, self.beta1, self.beta2, self.eps, self.t = torch, lr, beta1, beta2, eps, 0
        self.m = [torch.zeros(st.n, dtype=torch.float64, device=st.dev) for st in states]
        self.v = [torch.zeros(st.n, dtype=torch.float64, device=st.dev) for st in states]

    def step(self, states, grads):
        self.t += 1
        bc1, bc2 = 1 - self.beta1 ** self.t, 1 - self.beta2 ** self.t  # host f64, as the reference
        for st, g, m, v in zip(states, grads, self.m, self.v):
            _lib.check(_lib.lib().mesw_adam_step(st.steps.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), st.n,
                                                 self.lr, self.beta1, self.beta2, self.eps, bc1, bc2,
                                                 C.c_float(STEP_FLOOR), _stream(self.torch, st.dev)))


class _Model:
    """Frozen base weights + per-layer effective-weight buffers on the device."""

    def __init__(self, torch, model, dev):
        mats = [model.embedding, *model.layers, model.head]
        self.base = [torch.as_tensor(np.asarray(w, np.float32)).to(dev).contiguous() for w in mats]
        self.eff = [torch.empty_like(w) for w in self.base]
        self.depth = len(mats) - 2
        self.vocab, self.width = self.base[0].shape


def _check_ids(vocab, seq):
    ids = np.asarray(seq, dtype=np.int64)
    if ids.ndim != 1 or ids.size == 0:
        raise ValueError("token sequence must be non-empty and 1-D")
    if ids.min() < 0 or ids.max() >= vocab:
        raise ValueError(f"token id out of range [0, {vocab})")
    return ids


def _teacher_logits(torch, ft: _Model, seq, dev):
    """toylm.forward (toylm.py:162-168) of the fine-tuned model."""
    ids = torch.from_numpy(_check_ids(ft.vocab, seq)).to(dev)
    h = ft.base[0][ids] + torch.from_numpy(_positional_bias(ids.numel(), ft.width)).to(dev)
    for w in ft.base[1:1 + ft.depth]:
        h = torch.clamp_min(h @ w, 0.0)
    return h @ ft.base[-1]


def backward_step_sizes(torch, base: _Model, states, sequences, targets, dev):
    """toylm.backward_step_sizes (toylm.py:394-447) -> (per-layer step grads, loss)."""
    if len(states) != base.depth + 2:
        raise ValueError(f"expected {base.depth + 2} layer states, got {len(states)}")
    ids_np = np.concatenate([_check_ids(base.vocab, s) for s in sequences])
    ids = torch.from_numpy(ids_np).to(dev)
    tgt = torch.cat(targets, dim=0)
    pos = torch.from_numpy(np.concatenate([_positional_bias(len(s), base.width) for s in sequences], axis=0)).to(dev)
    mats = [st.effective(bw, ew) for st, bw, ew in zip(states, base.base, base.eff)]
    h = mats[0][ids] + pos
    pre, acts = [], [h]
    for w in mats[1:1 + base.depth]:
        z = acts[-1] @ w
        pre.append(z)
        acts.append(torch.clamp_min(z, 0.0))
    logits = acts[-1] @ mats[-1]
    if logits.shape != tgt.shape:
        raise ValueError(f"target logits shape {tuple(tgt.shape)} != model logits shape {tuple(logits.shape)}")
    diff = logits.double() - tgt.double()
    loss = float((diff * diff).mean())
    grads = [None] * len(states)
    g_logits = (2.0 * diff / diff.numel()).float()
    grads[-1] = states[-1].step_gradient(acts[-1].T @ g_logits)
    g_h = g_logits @ mats[-1].T
    for li in range(base.depth, 0, -1):
        g_z = torch.where(pre[li - 1] > 0.0, g_h, torch.zeros((), dtype=g_h.dtype, device=dev))
        grads[li] = states[li].step_gradient(acts[li - 1].T @ g_z)
        g_h = g_z @ mats[li].T
    up = torch.zeros_like(states[0].delta)
    up.index_add_(0, ids, g_h)
    grads[0] = states[0].step_gradient(up)
    return grads, loss


def _repack(torch, art, st: _LayerState):
    """compress._repack (compress.py:325-335) with mesw_quantize_pack."""
    L = _lib.lib()
    packed = torch.empty(int(L.mesw_packed_nbytes(st.m, st.n, st.bits)), dtype=torch.uint8, device=st.dev)
    _lib.check(L.mesw_quantize_pack(st.delta.data_ptr(), st.m, st.n, st.steps.data_ptr(), st.bits,
                                    st.mask.data_ptr(), packed.data_ptr(), _stream(torch, st.dev)))
    steps = st.steps.cpu().numpy().copy()
    return replace(art, steps=steps, packed=PackedCodes(bits=st.bits, rows=st.m, cols=st.n,
                                                        data=packed.cpu().numpy().tobytes()))


def distill_step_sizes(base, finetuned, artifacts, sequences, cfg: DistillConfig = DistillConfig(),
                       device="cuda") -> DistillResult:
    """compress.distill_step_sizes (compress.py:331-378): train the step sizes of
    `artifacts` (one CompressedDelta per weight layer: embedding, hidden..., head) so the
    base + compressed deltas match the fine-tuned model's logits on `sequences`.
    `base` / `finetuned` expose `embedding`, `layers`, `head` (toylm.ToyLM or alike)."""
    import torch
    if not sequences:
        raise ValueError("calibration set is empty")
    dev = torch.device(device)
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # f32 GEMMs, as the reference's numpy
    try:
        bm, fm = _Model(torch, base, dev), _Model(torch, finetuned, dev)
        if len(artifacts) != bm.depth + 2:
            raise ValueError(f"expected {bm.depth + 2} layer artifacts, got {len(artifacts)}")
        states = [_LayerState(torch, fw - bw, art, dev) for bw, fw, art in zip(bm.base, fm.base, artifacts)]
        targets = [_teacher_logits(torch, fm, s, dev) for s in sequences]
        _, initial = backward_step_sizes(torch, bm, states, sequences, targets, dev)
        opt = _Adam(torch, states, cfg.lr)
        batch_losses = []
        for _ in range(cfg.epochs):
            for s0 in range(0, len(sequences), cfg.batch_size):
                grads, loss = backward_step_sizes(torch, bm, states, sequences[s0:s0 + cfg.batch_size],
                                                  targets[s0:s0 + cfg.batch_size], dev)
                batch_losses.append(loss)
                if initial > 0 and loss > 10.0 * initial:
                    raise DistillDivergenceError(f"batch loss {loss:.6g} exceeded 10x initial loss {initial:.6g}")
                opt.step(states, grads)
        _, final = backward_step_sizes(torch, bm, states, sequences, targets, dev)
        layers = [_repack(torch, art, st) for art, st in zip(artifacts, states)]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    return DistillResult(layers=layers, initial_loss=initial, final_loss=final, batch_losses=batch_losses)
