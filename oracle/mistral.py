"""Oracle for the Mistral-shaped multi-expert decode step (numpy, f32/f64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The reference toy model has
no attention (toylm.py:1-8); this restates the standard Mistral decoder step
around Eq. 4 linears: y = x.W + x.reconstruct_e() per projection
(compress.py:115-121), with RMSNorm, rotate-half RoPE,
GQA attention over a KV cache, SwiGLU and greedy argmax (toylm.py:247).
"""

from __future__ import annotations

import numpy as np


def rmsnorm(x, w, eps):
    x = x.astype(np.float64)
    return (x / np.sqrt((x * x).mean(-1, keepdims=True) + eps)) * w.astype(np.float64)


def rope(v, pos, theta):
    """v: [heads, D] for one token at position pos (rotate-half convention)."""
    D = v.shape[-1]
    half = D // 2
    inv = theta ** (-2.0 * np.arange(half) / D)
    ang = pos * inv
    c, s = np.cos(ang), np.sin(ang)
    x0, x1 = v[..., :half], v[..., half:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)


def decode_step(shape, weights, deltas, kcache, vcache, ids, pos, expert_of):
    """One step for B requests.

    weights: dict(embedding [V,H], final_norm [H], head [H,V], layers=[dict(attn_norm, q,k,v,o,
             mlp_norm, gate, up, down)]) as float arrays (already bf16-rounded by the caller).
    deltas:  deltas[slot][layer][proj] = dense f32 delta [in, out] (or missing for no delta).
    kcache/vcache: [L][B][ctx][n_kv][D] float arrays (positions < pos valid); updated in place.
    expert_of[b] = slot or -1.  Returns (logits [B,V] f64, next ids [B]).
    """
    s = shape
    H, D, nh, nkv = s.hidden, s.head_dim, s.n_heads, s.n_kv_heads
    G = nh // nkv
    B = len(ids)
    h = weights["embedding"][np.asarray(ids)].astype(np.float64)

    def lin(x, l, name, b):
        y = x @ weights["layers"][l][name].astype(np.float64)
        e = expert_of[b]
        if e >= 0 and name in deltas[e][l]:
            y = y + x @ deltas[e][l][name].astype(np.float64)
        return y

    for l, lw in enumerate(weights["layers"]):
        for b in range(B):
            x = rmsnorm(h[b], lw["attn_norm"], s.rms_eps)
            q = lin(x, l, "q", b).reshape(nh, D)
            k = lin(x, l, "k", b).reshape(nkv, D)
            v = lin(x, l, "v", b).reshape(nkv, D)
            p = int(pos[b])
            q = rope(q, p, s.rope_theta)
            k = rope(k, p, s.rope_theta)
            kcache[l][b][p] = k
            vcache[l][b][p] = v
            K = kcache[l][b][:p + 1].astype(np.float64)  # [T, nkv, D]
            V = vcache[l][b][:p + 1].astype(np.float64)
            out = np.zeros((nh, D))
            for hh in range(nh):
                g = hh // G
                sc = (K[:, g, :] @ q[hh]) / np.sqrt(D)
                sc = np.exp(sc - sc.max())
                sc /= sc.sum()
                out[hh] = sc @ V[:, g, :]
            h[b] = h[b] + lin(out.reshape(-1), l, "o", b)
            x = rmsnorm(h[b], lw["mlp_norm"], s.rms_eps)
            gt = lin(x, l, "gate", b)
            up = lin(x, l, "up", b)
            act = gt / (1.0 + np.exp(-gt)) * up
            h[b] = h[b] + lin(act, l, "down", b)
    x = rmsnorm(h, weights["final_norm"], s.rms_eps)
    logits = x @ weights["head"].astype(np.float64)
    return logits, np.argmax(logits, axis=-1)
