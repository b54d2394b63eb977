"""Host-side mirror of the reference's quantizer types (quant.py:39-61, :172-192).

Only the metadata the serving path needs lives here: the code range, the packed
container type and its byte arithmetic.  Decoding codes happens on the GPU
(`device.DeviceDelta`), see `csrc/mesw_repack.cu`.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib

__all__ = ["QuantConfig", "PackedCodes", "packed_nbytes", "ALLOWED_BITS"]

ALLOWED_BITS = (1, 2, 3, 4, 8)


@dataclass(frozen=True)
class QuantConfig:
    """Bit width and derived code range (quant.py:39-61)."""

    bits: int = 2

    def __post_init__(self):
        if self.bits not in ALLOWED_BITS:
            raise ValueError(f"bits must be one of {ALLOWED_BITS}, got {self.bits}")

    @property
    def q_n(self) -> int:
        return 1 if self.bits == 1 else 2 ** (self.bits - 1)

    @property
    def q_p(self) -> int:
        return 1 if self.bits == 1 else 2 ** (self.bits - 1) - 1


@dataclass(frozen=True)
class PackedCodes:
    """Column-major bit-packed offset codes (quant.py:172-187)."""

    bits: int
    rows: int
    cols: int
    data: bytes

    @property
    def bytes_per_col(self) -> int:
        return (self.rows * self.bits + 7) // 8


def packed_nbytes(rows: int, cols: int, bits: int) -> int:
    """quant.packed_nbytes (quant.py:190-192), computed by the C ABI."""
    return int(_lib.lib().mesw_packed_nbytes(rows, cols, bits))
