"""CPU restatement of the reference's layer compression (TEST INFRASTRUCTURE ONLY).

Follows compress.compress_layer (compress.py:178-215) for the default metric
("reconstruction"): quant.init_step_sizes (quant.py:81-99), quant.quantize_codes
(quant.py:111-120, f64 division, round-half-away-from-zero), quant.dequantize
(quant.py:135-139), salient.score_reconstruction (salient.py:106-120, f64 row error),
salient.top_k (salient.py:141-151, stable argsort), fp16 salient rows (compress.py:208-209)
and quant.pack_codes (quant.py:195-213).  Pinned against the reference's own
compress_layer artifacts in tests/golden (layer_*.mesw with their inputs in
layer_expected.npz).

The summation orders the GPU kernels reproduce are those of these numpy calls:
`((a - b) ** 2).sum(axis=1)` on a C-contiguous f64 array is numpy's pairwise sum per row
(`pairwise_sum_f64` below restates it); `np.abs(x).mean(axis=0, dtype=float64)` on f32
accumulates rows sequentially in f64.
"""

from __future__ import annotations

import numpy as np

from .mesw import OracleLayer, code_range, pack_codes

TINY_F32 = np.float32(1.1754944e-38)  # numerics.py:26


def pairwise_sum_f64(a: np.ndarray) -> float:
    """numpy's pairwise summation of a contiguous f64 vector (8-way unrolled blocks of
    <= 128, halving split rounded down to a multiple of 8)."""
    def rec(lo, n):
        if n < 8:
            res = 0.0
            for i in range(n):
                res += a[lo + i]
            return res
        if n <= 128:
            r = [float(a[lo + j]) for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)
    return rec(0, a.shape[0])


def init_step_sizes(x: np.ndarray, bits: int) -> np.ndarray:
    """quant.py:81-99."""
    x = np.asarray(x, dtype=np.float32)
    q_n, q_p = code_range(bits)
    if x.shape[0] == 0:
        raw = np.zeros(x.shape[1], dtype=np.float64)
    elif bits == 1:
        raw = np.abs(x).mean(axis=0, dtype=np.float64)
    else:
        raw = np.abs(x).max(axis=0).astype(np.float64) / q_p
    steps = raw.astype(np.float32)
    steps[raw <= 0.0] = TINY_F32
    return steps


def quantize_codes(x: np.ndarray, steps: np.ndarray, bits: int) -> np.ndarray:
    """quant.py:111-120."""
    x = np.asarray(x, dtype=np.float32)
    if bits == 1:
        return np.where(x < 0, -1, 1).astype(np.int8)
    q_n, q_p = code_range(bits)
    u = x.astype(np.float64) / steps.astype(np.float64)
    return np.clip(np.copysign(np.floor(np.abs(u) + 0.5), u), -q_n, q_p).astype(np.int8)


def compress_layer(delta: np.ndarray, energy: np.ndarray, bits: int, k: int) -> OracleLayer:
    """compress.py:178-215 with metric "reconstruction"."""
    delta = np.asarray(delta, dtype=np.float32)
    m, n = delta.shape
    if k > m:
        raise ValueError("salient_k exceeds the input channels")
    steps0 = init_step_sizes(delta, bits)
    approx0 = (quantize_codes(delta, steps0, bits).astype(np.float32) * steps0[None, :]).astype(np.float32)
    row_err = ((delta.astype(np.float64) - approx0.astype(np.float64)) ** 2).sum(axis=1)
    scores = (np.asarray(energy, np.float32).astype(np.float64) * row_err).astype(np.float32)
    order = np.argsort(-scores, kind="stable")[:k]
    idx = np.sort(order).astype(np.int64)
    mask = np.ones(m, dtype=bool)
    mask[idx] = False
    steps = init_step_sizes(delta[mask], bits)
    codes = np.zeros((m, n), dtype=np.int8)
    if mask.any():
        codes[mask] = quantize_codes(delta[mask], steps, bits)
    with np.errstate(over="ignore"):
        rows = delta[idx].astype(np.float16)
    return OracleLayer(m, n, bits, k, idx, rows, steps, pack_codes(codes, bits))
