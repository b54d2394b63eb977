"""Deterministic synthetic Mistral-7B-shaped workloads (no network, random init).

Synthetic compressed deltas follow SURVEY.md §8(d): at b=2 every byte string is a
valid code stream, so codes are random bytes with the salient rows' codes forced
to offset Q_N (q = 0, as compress_layer writes them, compress.py:205-214); steps
|N(0,1e-3)|+1e-6; 8 salient input channels; salient rows N(0, 0.02) in fp16.
Artifacts are real MESW containers (serialize_artifact) so the bench exercises
the same loader path as reference-produced files.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .compress import (ArtifactManifest, CompressedDelta, ExpertArtifact, SalientSet,
                       serialize_artifact)
from .quant import PackedCodes


@dataclass(frozen=True)
class MistralShape:
    """Mistral-7B decoder geometry (PAPER.md:406 uses Mistral-7B experts)."""

    hidden: int = 4096
    intermediate: int = 14336
    n_layers: int = 32
    n_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    vocab: int = 32000
    rope_theta: float = 1e6
    rms_eps: float = 1e-5

    @property
    def proj_shapes(self) -> list:
        """(name, m_in, n_out) of the 7 compressed linears of one decoder layer."""
        h, i, kv = self.hidden, self.intermediate, self.n_kv_heads * self.head_dim
        return [("q", h, h), ("k", h, kv), ("v", h, kv), ("o", h, h),
                ("gate", h, i), ("up", h, i), ("down", i, h)]


def synthetic_layer(rng: np.random.Generator, m: int, n: int, k: int = 8, bits: int = 2) -> CompressedDelta:
    """One synthetic 2-bit compressed layer block (column-major packed codes)."""
    if bits != 2:
        raise NotImplementedError("synthetic fast path is defined for b=2")
    bpc = (m * 2 + 7) // 8
    runs = np.frombuffer(rng.bytes(n * bpc), dtype=np.uint8).reshape(n, bpc).copy()
    if m % 4:
        # zero the padding bits of the last byte of each run (pack_codes pads with 0)
        valid = (m % 4) * 2
        runs[:, -1] &= np.uint8((1 << valid) - 1)
    idx = np.sort(rng.choice(m, size=k, replace=False)).astype(np.int64)
    for i in idx:  # offset 2 (0b10) = q 0 in every column
        byte, sh = i // 4, (i % 4) * 2
        runs[:, byte] = (runs[:, byte] & np.uint8(~(3 << sh) & 0xFF)) | np.uint8(2 << sh)
    steps = (np.abs(rng.normal(0.0, 1e-3, size=n)) + 1e-6).astype(np.float32)
    rows = rng.normal(0.0, 0.02, size=(k, n)).astype(np.float16)
    return CompressedDelta(salient=SalientSet(indices=idx, k=k), salient_rows=rows, steps=steps,
                           packed=PackedCodes(bits=2, rows=m, cols=n, data=runs.tobytes()))


def synthetic_expert_artifact(seed: int, shapes: list, domain: str, k: int = 8) -> bytes:
    """Serialized MESW artifact with one block per (m, n) in `shapes`."""
    layers = []
    for li, (m, n) in enumerate(shapes):
        rng = np.random.default_rng(np.random.SeedSequence((seed, li)))
        layers.append(synthetic_layer(rng, m, n, k))
    man = ArtifactManifest(model_id=f"synthetic-{domain}-{seed}", domain=domain,
                           base_digest="synthetic", layer_count=len(layers))
    return serialize_artifact(ExpertArtifact(manifest=man, layers=layers))


def mistral_expert_shapes(shape: MistralShape = MistralShape(), n_layers: int | None = None) -> list:
    """Block shapes of a Mistral expert artifact: 7 projections per decoder layer."""
    L = shape.n_layers if n_layers is None else n_layers
    return [(m, n) for _ in range(L) for (_, m, n) in shape.proj_shapes]


def linear_bytes(m: int, n: int, n_experts: int, B: int, k: int = 8, base: bool = True) -> int:
    """Algorithmic HBM bytes of one fused multi-expert decode linear:
    bf16 base + per expert (2-bit codes + fp16 salient rows + f32 steps + u32 idx)
    + bf16 x in + bf16 y out."""
    per_expert = m * n // 4 + 2 * k * n + 4 * n + 4 * k
    return (2 * m * n if base else 0) + n_experts * per_expert + 2 * B * m + 2 * B * n
