"""Oracle restatement of the toy-model forward with delta providers and the
SPEC's batched multi-model forward.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Lets the GPU tests run the
reference's provider protocol on the GPU box, where /root/reference is absent.
"""

from __future__ import annotations

import numpy as np

from .mesw import OracleLayer


def positional_bias(n_positions: int, width: int) -> np.ndarray:
    """Sinusoidal table, toylm.py:87-93."""
    pos = np.arange(n_positions, dtype=np.float64)[:, None]
    dim = np.arange(width, dtype=np.float64)[None, :]
    angle = pos / np.power(10000.0, (2.0 * (dim // 2)) / width)
    return np.where(dim % 2 == 0, np.sin(angle), np.cos(angle)).astype(np.float32)


class ToyWeights:
    """Plain container: embedding [V,d], hidden layers [d,d]..., head [d,V] (toylm.py:46-74)."""

    def __init__(self, embedding, layers, head):
        self.embedding = np.asarray(embedding, np.float32)
        self.layers = [np.asarray(w, np.float32) for w in layers]
        self.head = np.asarray(head, np.float32)
        self.vocab, self.width = self.embedding.shape
        self.depth = len(self.layers)

    @property
    def n_weight_layers(self) -> int:
        return self.depth + 2

    def weight_matrices(self):
        return [self.embedding, *self.layers, self.head]


class DenseProvider:
    """Exact provider over a dense delta (SPEC.md:414 `Exact`)."""

    def __init__(self, dense: np.ndarray):
        self.dense = np.asarray(dense, np.float32)

    def matvec_batch(self, h):
        return np.asarray(h, np.float32) @ self.dense

    def matvec(self, x):
        return np.asarray(x, np.float32) @ self.dense

    def rows(self, ids):
        return self.dense[np.asarray(ids, np.int64)]

    def row(self, i):
        return self.dense[int(i)]


class OracleCompressedProvider(DenseProvider):
    """Provider backed by oracle reconstruct() of one compressed layer."""

    def __init__(self, layer: OracleLayer):
        super().__init__(layer.reconstruct())


def _check_tokens(model: ToyWeights, tokens) -> np.ndarray:
    ids = np.asarray(tokens, dtype=np.int64)
    if ids.ndim != 1 or ids.size == 0:
        raise ValueError("token sequence must be non-empty and 1-D")
    if ids.min() < 0 or ids.max() >= model.vocab:
        raise ValueError("token id out of range")
    return ids


def _provider_rows(provider, ids, cols):
    """toylm.py:171-180: None -> zeros; `rows(ids)` if present, else per-id `row(i)`."""
    if provider is None:
        return np.zeros((ids.size, cols), np.float32)
    if hasattr(provider, "rows"):
        return np.asarray(provider.rows(ids), np.float32)
    return np.stack([np.asarray(provider.row(int(t)), np.float32) for t in ids])


def _apply_delta(h, provider):
    """toylm.py:183-186: prefer matvec_batch, else per-row matvec."""
    if hasattr(provider, "matvec_batch"):
        return np.asarray(provider.matvec_batch(h), np.float32)
    return np.stack([np.asarray(provider.matvec(r), np.float32) for r in h])


def forward_with_delta(base: ToyWeights, providers, tokens) -> np.ndarray:
    """toylm.py:189-211."""
    if len(providers) != base.n_weight_layers:
        raise ValueError(f"expected {base.n_weight_layers} delta providers, got {len(providers)}")
    ids = _check_tokens(base, tokens)
    h = base.embedding[ids] + positional_bias(ids.size, base.width)
    h = h + _provider_rows(providers[0], ids, base.width)
    for w, p in zip(base.layers, providers[1:-1]):
        z = h @ w
        if p is not None:
            z = z + _apply_delta(h, p)
        h = np.maximum(z, 0.0)
    logits = h @ base.head
    if providers[-1] is not None:
        logits = logits + _apply_delta(h, providers[-1])
    return logits


def forward(base: ToyWeights, tokens) -> np.ndarray:
    """toylm.py:162-168."""
    return forward_with_delta(base, [None] * base.n_weight_layers, tokens)


def greedy_decode(base: ToyWeights, prompt, max_new: int, providers=None) -> list[int]:
    """toylm.py:234-248 (single-position steps; argmax = first maximum)."""
    ids = list(_check_tokens(base, prompt))
    provs = providers if providers is not None else [None] * base.n_weight_layers
    if len(provs) != base.n_weight_layers:
        raise ValueError("provider count mismatch")
    for _ in range(max_new):
        pos = len(ids) - 1
        tok = np.asarray([ids[-1]], np.int64)
        h = base.embedding[tok] + positional_bias(pos + 1, base.width)[pos:pos + 1]
        h = h + _provider_rows(provs[0], tok, base.width)
        for w, p in zip(base.layers, provs[1:-1]):
            z = h @ w
            if p is not None:
                z = z + _apply_delta(h, p)
            h = np.maximum(z, 0.0)
        logits = h @ base.head
        if provs[-1] is not None:
            logits = logits + _apply_delta(h, provs[-1])
        ids.append(int(np.argmax(logits[0])))
    return ids


def batched_multi_model_forward(base: ToyWeights, experts: dict, plan) -> list:
    """SPEC.md:433-438 restated: per query (qid, expert, tokens) -> logits or error entry.

    ``experts`` maps expert id -> provider list.  Unknown expert -> ("error", msg)
    for that query; the rest of the batch continues.
    """
    out = []
    for qid, eid, toks in plan:
        if eid not in experts:
            out.append((qid, None, f"unknown expert {eid!r}"))
            continue
        out.append((qid, forward_with_delta(base, experts[eid], toks), None))
    return out
