"""Oracle restatement of the MESW container, code layout and Eq. 4 delta math.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Reference citations are
into /root/reference/pkg/src/meswitch/ unless marked SPEC.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass

import numpy as np

TINY_F32 = float(np.finfo(np.float32).tiny)  # numerics.py:26
MAGIC = b"MESW"  # compress.py:60
VERSION = 1  # compress.py:61


class OracleArtifactError(Exception):
    """Mirror of errors.ArtifactError (errors.py:19)."""


class OracleBadMagic(OracleArtifactError):
    pass


class OracleUnsupportedVersion(OracleArtifactError):
    pass


class OracleTruncated(OracleArtifactError):
    pass


# --------------------------------------------------------------------------
# quant.py code range and packing
# --------------------------------------------------------------------------

def code_range(bits: int) -> tuple[int, int]:
    """(Q_N, Q_P) -- quant.py:49-61.  1-bit codes are +-1."""
    if bits not in (1, 2, 3, 4, 8):
        raise ValueError(f"bits must be one of (1, 2, 3, 4, 8), got {bits}")
    if bits == 1:
        return 1, 1
    return 1 << (bits - 1), (1 << (bits - 1)) - 1


def bytes_per_col(rows: int, bits: int) -> int:
    """quant.py:186-187."""
    return (rows * bits + 7) // 8


def packed_nbytes(rows: int, cols: int, bits: int) -> int:
    """quant.py:190-192."""
    return cols * bytes_per_col(rows, bits)


def unpack_codes(data: bytes, rows: int, cols: int, bits: int) -> np.ndarray:
    """Decode a column-major LSB-first offset-code stream to int8 codes [rows, cols].

    Follows quant.py:216-236: column j owns bytes [j*bpc, (j+1)*bpc); row i's
    offset occupies bits [i*b, i*b+b) of that run, little-endian bit order;
    q = u - Q_N for b>=2 and q = 2u - 1 for b=1.  Implemented with a two-byte
    window per value (a b<=8 value spans at most two bytes).
    """
    expected = packed_nbytes(rows, cols, bits)
    if len(data) != expected:
        raise ValueError(f"packed stream has {len(data)} bytes, expected {expected}")
    q_n, _ = code_range(bits)
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dtype=np.int8)
    bpc = bytes_per_col(rows, bits)
    if bits == 2:  # byte-aligned fields: 4 codes per byte, LSB first (same result, vectorised)
        run = np.frombuffer(data, dtype=np.uint8).reshape(cols, bpc)
        u = np.empty((cols, bpc, 4), dtype=np.int8)
        for f in range(4):
            u[:, :, f] = (run >> np.uint8(2 * f)) & np.uint8(3)
        q = u.reshape(cols, 4 * bpc)[:, :rows] - np.int8(q_n)
        return np.ascontiguousarray(q.T)
    runs = np.zeros((cols, bpc + 1), dtype=np.uint16)
    runs[:, :bpc] = np.frombuffer(data, dtype=np.uint8).reshape(cols, bpc)
    bit_off = np.arange(rows, dtype=np.int64) * bits
    lo = bit_off >> 3
    sh = (bit_off & 7).astype(np.uint16)
    window = runs[:, lo] | (runs[:, lo + 1] << np.uint16(8))  # [cols, rows]
    u = ((window >> sh[None, :]) & np.uint16((1 << bits) - 1)).astype(np.int16)
    q = (2 * u - 1) if bits == 1 else (u - q_n)
    return np.ascontiguousarray(q.T.astype(np.int8))


def _unpack_window(data: bytes, rows: int, cols: int, bits: int) -> np.ndarray:
    """Decode a column-major LSB-first offset-code stream to int8 codes [rows, cols].

    Follows quant.py:216-236: column j owns bytes [j*bpc, (j+1)*bpc); row i's
    offset occupies bits [i*b, i*b+b) of that run, little-endian bit order;
    q = u - Q_N for b>=2 and q = 2u - 1 for b=1.  Implemented with a two-byte
    window per value (a b<=8 value spans at most two bytes).
    """
    expected = packed_nbytes(rows, cols, bits)
    if len(data) != expected:
        raise ValueError(f"packed stream has {len(data)} bytes, expected {expected}")
    q_n, _ = code_range(bits)
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dtype=np.int8)
    bpc = bytes_per_col(rows, bits)
    runs = np.zeros((cols, bpc + 1), dtype=np.uint16)
    runs[:, :bpc] = np.frombuffer(data, dtype=np.uint8).reshape(cols, bpc)
    bit_off = np.arange(rows, dtype=np.int64) * bits
    lo = bit_off >> 3
    sh = (bit_off & 7).astype(np.uint16)
    window = runs[:, lo] | (runs[:, lo + 1] << np.uint16(8))  # [cols, rows]
    u = ((window >> sh[None, :]) & np.uint16((1 << bits) - 1)).astype(np.int16)
    q = (2 * u - 1) if bits == 1 else (u - q_n)
    return np.ascontiguousarray(q.T.astype(np.int8))


def pack_codes(codes: np.ndarray, bits: int) -> bytes:
    """Inverse of unpack_codes (quant.py:195-213), used to build test artifacts."""
    codes = np.asarray(codes)
    rows, cols = codes.shape
    q_n, q_p = code_range(bits)
    if bits == 1:
        if not np.isin(codes, (-1, 1)).all():
            raise ValueError("1-bit codes must be -1 or +1")
        u = ((codes.astype(np.int16) + 1) // 2).astype(np.uint32)
    else:
        if codes.size and (codes.min() < -q_n or codes.max() > q_p):
            raise ValueError("codes out of range")
        u = (codes.astype(np.int16) + q_n).astype(np.uint32)
    if rows == 0 or cols == 0:
        return b""
    bpc = bytes_per_col(rows, bits)
    out = np.zeros((cols, bpc + 1), dtype=np.uint32)
    for i in range(rows):  # per-row scatter of b-bit fields into the run
        off = i * bits
        lo, sh = off >> 3, off & 7
        val = u[i, :] << np.uint32(sh)
        out[:, lo] |= val & 0xFF
        out[:, lo + 1] |= (val >> 8) & 0xFF
    return out[:, :bpc].astype(np.uint8).tobytes()


# --------------------------------------------------------------------------
# compress.py CompressedDelta / reconstruct
# --------------------------------------------------------------------------

@dataclass
class OracleLayer:
    """One layer block of an MESW artifact (compress.py:87-121 field set)."""

    m: int
    n: int
    bits: int
    k: int
    salient_idx: np.ndarray  # int64[k], strictly ascending (salient.py:46-57)
    salient_rows: np.ndarray  # float16[k, n]
    steps: np.ndarray  # float32[n]
    packed: bytes

    def codes(self) -> np.ndarray:
        return unpack_codes(self.packed, self.m, self.n, self.bits)

    def unpack_generic(self) -> np.ndarray:
        """The two-byte-window decode for every width (pins the vectorised 2-bit path)."""
        return _unpack_window(self.packed, self.m, self.n, self.bits)

    def reconstruct(self) -> np.ndarray:
        """Dense f32 delta: codes*steps, salient rows overwritten (compress.py:115-121)."""
        q = self.codes().astype(np.float32)
        out = (q * self.steps.astype(np.float32)[None, :]).astype(np.float32)
        if self.k:
            out[self.salient_idx] = self.salient_rows.astype(np.float32)
        return out


def delta_matvec_batch(x: np.ndarray, layer: OracleLayer, dense: np.ndarray | None = None) -> np.ndarray:
    """SPEC.md:424-432 delta_matvec for a batch of rows, computed in float64.

    y_j = s_j * sum_{i not salient} x_i q_ij + sum_{i salient} x_i * half(R_i)_j.
    If ``dense`` (a reconstruct()) is supplied it is used instead, which is the
    dequantize-then-matvec reference the SPEC compares against.
    """
    x = np.asarray(x, dtype=np.float64)
    if dense is not None:
        return x @ dense.astype(np.float64)
    q = layer.codes().astype(np.float64)
    if layer.k:
        q[layer.salient_idx] = 0.0
    y = (x @ q) * layer.steps.astype(np.float64)[None, :]
    if layer.k:
        y += x[:, layer.salient_idx] @ layer.salient_rows.astype(np.float64)
    return y


# --------------------------------------------------------------------------
# MESW container (compress.py:481-559)
# --------------------------------------------------------------------------

def parse_artifact(data: bytes) -> tuple[dict, list[OracleLayer]]:
    """Restatement of deserialize_artifact (compress.py:513-549)."""
    pos = 0

    def take(nb: int) -> bytes:
        nonlocal pos
        if pos + nb > len(data):
            raise OracleTruncated(f"need {nb} bytes at offset {pos}")
        chunk = data[pos:pos + nb]
        pos += nb
        return chunk

    if take(4) != MAGIC:
        raise OracleBadMagic("bad magic")
    (version,) = struct.unpack("<H", take(2))
    if version != VERSION:
        raise OracleUnsupportedVersion(f"version {version}")
    (mlen,) = struct.unpack("<I", take(4))
    manifest = json.loads(take(mlen).decode("utf-8"))
    layers = []
    for _ in range(int(manifest["layer_count"])):
        m, n, bits, k = struct.unpack("<IIBI", take(13))
        idx = np.frombuffer(take(4 * k), dtype="<u4").astype(np.int64)
        rows = np.frombuffer(take(2 * k * n), dtype="<u2").reshape(k, n).view(np.float16).copy()
        steps = np.frombuffer(take(4 * n), dtype="<f4").astype(np.float32)
        (plen,) = struct.unpack("<I", take(4))
        if plen != packed_nbytes(m, n, bits):
            raise OracleTruncated("packed length mismatch")
        layers.append(OracleLayer(m, n, bits, k, idx, rows, steps, take(plen)))
    if pos != len(data):
        raise OracleTruncated("trailing bytes")
    return manifest, layers


def serialize_artifact(manifest: dict, layers: list[OracleLayer]) -> bytes:
    """Restatement of serialize_artifact (compress.py:481-495)."""
    out = bytearray(MAGIC)
    out += struct.pack("<H", VERSION)
    mj = json.dumps(manifest, sort_keys=True, separators=(",", ":")).encode("utf-8")
    out += struct.pack("<I", len(mj)) + mj
    for L in layers:
        out += struct.pack("<IIBI", L.m, L.n, L.bits, L.k)
        out += np.asarray(L.salient_idx, dtype="<u4").tobytes()
        out += np.asarray(L.salient_rows, dtype=np.float16).view("<u2").tobytes()
        out += np.asarray(L.steps, dtype="<f4").tobytes()
        out += struct.pack("<I", len(L.packed)) + L.packed
    return bytes(out)


def layer_block_nbytes(m: int, n: int, bits: int, k: int) -> int:
    """compress.py:589-597 total (header 13 + 4-byte packed prefix)."""
    return packed_nbytes(m, n, bits) + 2 * k * n + 4 * n + 4 * k + 17


# --------------------------------------------------------------------------
# Synthetic layers (test helpers; not reference code)
# --------------------------------------------------------------------------

def random_layer(rng: np.random.Generator, m: int, n: int, bits: int, k: int,
                 step_scale: float = 1e-3) -> OracleLayer:
    """A valid random compressed layer: random in-range codes, salient rows zeroed."""
    q_n, q_p = code_range(bits)
    if bits == 1:
        codes = rng.choice(np.array([-1, 1], dtype=np.int8), size=(m, n))
    else:
        codes = rng.integers(-q_n, q_p + 1, size=(m, n)).astype(np.int8)
    idx = np.sort(rng.choice(m, size=k, replace=False)).astype(np.int64) if k else np.zeros(0, np.int64)
    if k and bits != 1:
        codes[idx] = 0
    rows = rng.normal(0.0, 0.05, size=(k, n)).astype(np.float16)
    steps = (np.abs(rng.normal(0.0, step_scale, size=n)) + 1e-6).astype(np.float32)
    return OracleLayer(m, n, bits, k, idx, rows, steps, pack_codes(codes, bits))
