"""MESW artifact container: load / parse / size accounting (drop-in for the
reference's compress.py:87-121, :393-436, :481-607).

Parsing and validation run in the C ABI (`mesw_parse_header`,
`mesw_parse_layers`); this module turns the returned offsets into the same
dataclasses the reference exposes, as zero-copy numpy views of the file bytes.
Device upload lives in `device.py`.
"""

from __future__ import annotations

import ctypes as C
import json
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .quant import PackedCodes

__all__ = [
    "MAGIC",
    "VERSION",
    "SalientSet",
    "CompressedDelta",
    "ArtifactManifest",
    "ExpertArtifact",
    "LayerSizes",
    "SizeBreakdown",
    "deserialize_artifact",
    "serialize_artifact",
    "load_artifact",
    "save_artifact",
    "layer_block_nbytes",
    "compressed_size_bytes",
    "compress_layer",
]

MAGIC = b"MESW"
VERSION = 1


@dataclass(frozen=True)
class SalientSet:
    """Sorted unique salient input channels (salient.py:46-57)."""

    indices: np.ndarray
    k: int

    def __post_init__(self):
        if self.indices.shape != (self.k,):
            raise ValueError("index count must equal k")
        if self.k and (np.diff(self.indices) <= 0).any():
            raise ValueError("indices must be strictly ascending")


@dataclass(frozen=True)
class CompressedDelta:
    """One layer's compressed delta (compress.py:87-121): packed codes, per-output
    step sizes and fp16 salient rows.  `rows`/`cols` keep the reference's int
    properties; the GPU provider protocol lives in `infer.GpuCompressedProvider`."""

    salient: SalientSet
    salient_rows: np.ndarray  # (k, n) float16
    steps: np.ndarray  # (n,) float32
    packed: PackedCodes

    @property
    def rows(self) -> int:
        return self.packed.rows

    @property
    def cols(self) -> int:
        return self.packed.cols

    @property
    def bits(self) -> int:
        return self.packed.bits


@dataclass(frozen=True)
class ArtifactManifest:
    """compress.py:393-417."""

    model_id: str
    domain: str
    base_digest: str
    layer_count: int

    def to_json(self) -> bytes:
        payload = {"model_id": self.model_id, "domain": self.domain,
                   "base_digest": self.base_digest, "layer_count": self.layer_count}
        return json.dumps(payload, sort_keys=True, separators=(",", ":")).encode("utf-8")

    @classmethod
    def from_json(cls, raw: bytes) -> "ArtifactManifest":
        d = json.loads(raw.decode("utf-8"))
        return cls(model_id=d["model_id"], domain=d["domain"], base_digest=d["base_digest"],
                   layer_count=int(d["layer_count"]))


@dataclass(frozen=True)
class ExpertArtifact:
    manifest: ArtifactManifest
    layers: list

    def __post_init__(self):
        if len(self.layers) != self.manifest.layer_count:
            raise ValueError("manifest layer_count does not match layer blocks")


def deserialize_artifact(data: bytes) -> ExpertArtifact:
    """Parse an MESW container (compress.py:513-549) through the C ABI.

    Raises BadMagicError / UnsupportedVersionError / TruncatedArtifactError
    exactly where the reference does, including trailing bytes.
    """
    L = _lib.lib()
    data = bytes(data)
    buf = C.create_string_buffer(data, len(data)) if data else C.create_string_buffer(1)
    moff, mlen = C.c_uint64(), C.c_uint32()
    _lib.check(L.mesw_parse_header(buf, len(data), C.byref(moff), C.byref(mlen)))
    manifest = ArtifactManifest.from_json(data[moff.value:moff.value + mlen.value])
    count = manifest.layer_count
    views = (_lib.LayerView * max(count, 1))()
    _lib.check(L.mesw_parse_layers(buf, len(data), moff.value + mlen.value, count, views))
    arr = np.frombuffer(data, dtype=np.uint8)
    layers = []
    for v in views[:count]:
        idx = arr[v.idx_off:v.idx_off + 4 * v.k].view("<u4").astype(np.int64)
        rows = arr[v.rows_off:v.rows_off + 2 * v.k * v.n].view("<u2").reshape(v.k, v.n).view(np.float16)
        steps = arr[v.steps_off:v.steps_off + 4 * v.n].view("<f4").astype(np.float32)
        packed = PackedCodes(bits=v.bits, rows=v.m, cols=v.n,
                             data=data[v.codes_off:v.codes_off + v.codes_len])
        layers.append(CompressedDelta(salient=SalientSet(indices=idx, k=v.k), salient_rows=rows,
                                      steps=steps, packed=packed))
    return ExpertArtifact(manifest=manifest, layers=layers)


def serialize_artifact(artifact: ExpertArtifact) -> bytes:
    """MESW writer (compress.py:481-495); byte-identical to the reference."""
    out = bytearray(MAGIC)
    out += struct.pack("<H", VERSION)
    mj = artifact.manifest.to_json()
    out += struct.pack("<I", len(mj)) + mj
    for layer in artifact.layers:
        out += struct.pack("<IIBI", layer.rows, layer.cols, layer.bits, layer.salient.k)
        out += np.asarray(layer.salient.indices).astype("<u4").tobytes()
        out += np.asarray(layer.salient_rows, dtype=np.float16).view(np.uint16).astype("<u2").tobytes()
        out += np.asarray(layer.steps).astype("<f4").tobytes()
        out += struct.pack("<I", len(layer.packed.data)) + layer.packed.data
    return bytes(out)


def load_artifact(path) -> ExpertArtifact:
    with open(path, "rb") as f:
        return deserialize_artifact(f.read())


def save_artifact(artifact: ExpertArtifact, path) -> None:
    with open(path, "wb") as f:
        f.write(serialize_artifact(artifact))


LAYER_HEADER_BYTES = 13
PACKED_PREFIX_BYTES = 4


@dataclass(frozen=True)
class LayerSizes:
    codes: int
    salient_rows: int
    steps: int
    indices: int
    header: int

    @property
    def total(self) -> int:
        return self.codes + self.salient_rows + self.steps + self.indices + self.header


@dataclass(frozen=True)
class SizeBreakdown:
    file_header: int
    layers: list

    @property
    def total(self) -> int:
        return self.file_header + sum(layer.total for layer in self.layers)


def layer_block_nbytes(m: int, n: int, bits: int, k: int) -> LayerSizes:
    """Exact on-disk footprint of one layer block (compress.py:589-597)."""
    codes = int(_lib.lib().mesw_packed_nbytes(m, n, bits))
    return LayerSizes(codes=codes, salient_rows=2 * k * n, steps=4 * n, indices=4 * k,
                      header=LAYER_HEADER_BYTES + PACKED_PREFIX_BYTES)


def compressed_size_bytes(artifact: ExpertArtifact) -> SizeBreakdown:
    """compress.py:600-607."""
    fh = len(MAGIC) + 2 + 4 + len(artifact.manifest.to_json())
    return SizeBreakdown(file_header=fh, layers=[
        layer_block_nbytes(l.rows, l.cols, l.bits, l.salient.k) for l in artifact.layers])


def compress_layer(delta, stats, bits: int = 2, salient_k: int = 8, metric: str = "reconstruction",
                   device="cuda") -> CompressedDelta:
    """compress.compress_layer (compress.py:178-215) on the GPU, bit-exact with the
    reference for metric "reconstruction" (mesw_compress_layer, csrc/mesw_compress.cu).

    delta: f32 [m, n] (reference orientation: rows = input channels), numpy or torch;
    stats: ActivationStats-like (`.energy` f32 [m]) or the energy vector itself."""
    import torch
    if metric != "reconstruction":
        raise NotImplementedError("the GPU compressor implements the default 'reconstruction' metric")
    energy = getattr(stats, "energy", stats)
    if energy is None:
        raise ValueError("metric 'reconstruction' requires activation stats")
    dev = torch.device(device)
    d = torch.as_tensor(np.asarray(delta, np.float32) if not torch.is_tensor(delta) else delta).to(
        dev, torch.float32).contiguous()
    if d.ndim != 2:
        raise ValueError(f"expected a 2-D delta, got shape {tuple(d.shape)}")
    m, n = d.shape
    if salient_k > m:
        raise ValueError(f"salient_k={salient_k} exceeds {m} input channels")
    e = torch.as_tensor(np.asarray(energy, np.float32)).to(dev).contiguous()
    if e.shape != (m,):
        raise ValueError(f"stats cover {e.shape[0]} channels, delta has {m} rows")
    L = _lib.lib()
    steps = torch.empty(n, dtype=torch.float32, device=dev)
    idx = torch.empty(max(salient_k, 1), dtype=torch.int32, device=dev)
    rows = torch.empty((max(salient_k, 1), n), dtype=torch.int16, device=dev)
    packed = torch.empty(int(L.mesw_packed_nbytes(m, n, bits)), dtype=torch.uint8, device=dev)
    ws = torch.empty(int(L.mesw_compress_workspace_bytes(m, n)), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    _lib.check(L.mesw_compress_layer(d.data_ptr(), m, n, e.data_ptr(), bits, salient_k, steps.data_ptr(),
                                     idx.data_ptr(), rows.data_ptr(), packed.data_ptr(), ws.data_ptr(), ws.numel(),
                                     C.c_void_p(s.cuda_stream)))
    s.synchronize()
    k = salient_k
    return CompressedDelta(
        salient=SalientSet(indices=idx[:k].cpu().numpy().astype(np.int64), k=k),
        salient_rows=rows[:k].cpu().numpy().view(np.float16).reshape(k, n),
        steps=steps.cpu().numpy(),
        packed=PackedCodes(bits=bits, rows=m, cols=n, data=packed.cpu().numpy().tobytes()))
