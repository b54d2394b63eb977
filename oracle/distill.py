"""CPU restatement of the reference's step-size distillation (TEST INFRASTRUCTURE ONLY).

Follows compress.distill_step_sizes (compress.py:331-378): frozen base, fine-tuned
teacher logits, per-layer QuantizedLayerState (toylm.py:357-391) whose reconstruction
re-quantizes the raw delta at the current steps (salient rows fixed at their fp16
values), toylm.backward_step_sizes (toylm.py:394-447: f64 MSE over every logit,
exact linear / ReLU adjoints, straight-through quantizer), quant.ste_step_gradient
(quant.py:142-169), the AdamW-rule update (compress.py:276-302, f64 moments, weight
decay 0), the positive clamp STEP_FLOOR (compress.py:305) and the 10x divergence abort,
then _repack (compress.py:325-335: codes re-derived from the trained steps).
Pinned bit-for-bit against tests/golden/distill.npz (made by the reference itself).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .compress import quantize_codes
from .mesw import code_range
from .toylm import ToyWeights, positional_bias

STEP_FLOOR = 1e-8


def round_half_away(x):
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def ste_step_gradient(x, steps, bits, upstream):
    """quant.py:142-169."""
    x = np.asarray(x, np.float32)
    upstream = np.asarray(upstream, np.float32)
    if bits == 1:
        local = np.where(x < 0, -1.0, 1.0)
    else:
        q_n, q_p = code_range(bits)
        u = x.astype(np.float64) / np.asarray(steps, np.float32).astype(np.float64)
        local = round_half_away(u) - u
        local = np.where(u < -q_n, -float(q_n), local)
        local = np.where(u > q_p, float(q_p), local)
    return (upstream.astype(np.float64) * local).sum(axis=0).astype(np.float32)


@dataclass
class LayerState:
    """toylm.py:357-391."""
    delta: np.ndarray
    salient: np.ndarray
    salient_rows: np.ndarray  # f32 (fp16-rounded values)
    steps: np.ndarray
    bits: int

    def __post_init__(self):
        self.mask = np.ones(self.delta.shape[0], dtype=bool)
        self.mask[self.salient] = False

    def reconstruct(self):
        codes = quantize_codes(self.delta, self.steps, self.bits)
        approx = codes.astype(np.float32) * self.steps[None, :]  # quant.dequantize (f32 product)
        approx[~self.mask] = self.salient_rows
        return approx

    def step_gradient(self, upstream):
        masked = np.where(self.mask[:, None], upstream, 0.0)
        return ste_step_gradient(self.delta, self.steps, self.bits, masked)


def backward_step_sizes(base: ToyWeights, states, sequences, target_logits):
    """toylm.py:394-447."""
    ids = np.concatenate([np.asarray(s, np.int64) for s in sequences])
    targets = np.concatenate([np.asarray(t, np.float32) for t in target_logits])
    pos = np.concatenate([positional_bias(len(s), base.width) for s in sequences], axis=0)
    deltas = [st.reconstruct() for st in states]
    mats = [base.embedding + deltas[0]]
    mats += [w + d for w, d in zip(base.layers, deltas[1:-1])]
    mats.append(base.head + deltas[-1])
    h = mats[0][ids] + pos
    pre, acts = [], [h]
    for w in mats[1:1 + len(base.layers)]:
        z = acts[-1] @ w
        pre.append(z)
        acts.append(np.maximum(z, 0.0))
    logits = acts[-1] @ mats[-1]
    diff = logits.astype(np.float64) - targets.astype(np.float64)
    loss = float((diff * diff).mean())
    grads = [None] * len(states)
    g_logits = (2.0 * diff / diff.size).astype(np.float32)
    grads[-1] = states[-1].step_gradient(acts[-1].T @ g_logits)
    g_h = g_logits @ mats[-1].T
    for li in range(len(base.layers), 0, -1):
        g_z = np.where(pre[li - 1] > 0.0, g_h, 0.0)
        grads[li] = states[li].step_gradient(acts[li - 1].T @ g_z)
        g_h = g_z @ mats[li].T
    up = np.zeros_like(states[0].delta)
    np.add.at(up, ids, g_h)
    grads[0] = states[0].step_gradient(up)
    return grads, loss


class Adam:
    """compress.py:276-302."""

    def __init__(self, sizes, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.beta1, self.beta2, self.eps, self.t = lr, beta1, beta2, eps, 0
        self.m = [np.zeros(s, np.float64) for s in sizes]
        self.v = [np.zeros(s, np.float64) for s in sizes]

    def step(self, params, grads):
        self.t += 1
        out = []
        for i, (p, g) in enumerate(zip(params, grads)):
            g = g.astype(np.float64)
            self.m[i] = self.beta1 * self.m[i] + (1 - self.beta1) * g
            self.v[i] = self.beta2 * self.v[i] + (1 - self.beta2) * g * g
            m_hat = self.m[i] / (1 - self.beta1 ** self.t)
            v_hat = self.v[i] / (1 - self.beta2 ** self.t)
            out.append((p.astype(np.float64) - self.lr * m_hat / (np.sqrt(v_hat) + self.eps)).astype(np.float32))
        return out


def toy_forward(model: ToyWeights, tokens):
    ids = np.asarray(tokens, np.int64)
    h = model.embedding[ids] + positional_bias(ids.size, model.width)
    for w in model.layers:
        h = np.maximum(h @ w, 0.0)
    return h @ model.head


def distill_step_sizes(base: ToyWeights, finetuned: ToyWeights, init, sequences, epochs, lr, batch_size, bits=2):
    """compress.py:331-378.  init: per layer (salient idx, fp16 rows, steps).
    Returns (steps per layer, codes per layer, initial, final, batch_losses)."""
    mats_b = [base.embedding, *base.layers, base.head]
    mats_f = [finetuned.embedding, *finetuned.layers, finetuned.head]
    states = [LayerState((wf - wb).astype(np.float32), np.asarray(idx), np.asarray(rows, np.float16).astype(np.float32),
                         np.asarray(st, np.float32).copy(), bits)
              for wb, wf, (idx, rows, st) in zip(mats_b, mats_f, init)]
    targets = [toy_forward(finetuned, s) for s in sequences]
    _, initial = backward_step_sizes(base, states, sequences, targets)
    opt = Adam([st.steps.shape[0] for st in states], lr)
    losses = []
    for _ in range(epochs):
        for s0 in range(0, len(sequences), batch_size):
            grads, loss = backward_step_sizes(base, states, sequences[s0:s0 + batch_size], targets[s0:s0 + batch_size])
            losses.append(loss)
            if initial > 0 and loss > 10.0 * initial:
                raise RuntimeError("distillation diverged")
            for st, s in zip(states, opt.step([st.steps for st in states], grads)):
                st.steps = np.maximum(s, STEP_FLOOR).astype(np.float32)
    _, final = backward_step_sizes(base, states, sequences, targets)
    codes = []
    for st in states:
        c = np.zeros(st.delta.shape, np.int8)
        if st.mask.any():
            c[st.mask] = quantize_codes(st.delta[st.mask], st.steps, bits)
        codes.append(c)
    return [st.steps for st in states], codes, initial, final, losses
