"""Binary16 value type of the reference API (pkg/src/qqq/numerics.py:30-68).

Scalar helpers only (the carrier type for the bit-trick conversion API); the
array rounding used on the hot path is the device cvt.rn.f16.f64 in the CUDA
library.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["NAN_BITS", "Binary16", "encode_f16", "decode_f16"]

NAN_BITS = 0x7E00


@dataclass(frozen=True)
class Binary16:
    bits: int

    def __post_init__(self) -> None:
        if not 0 <= self.bits <= 0xFFFF:
            raise ValueError(f"binary16 pattern out of range: {self.bits:#x}")

    @classmethod
    def from_float(cls, x: float) -> "Binary16":
        return encode_f16(x)

    def to_float(self) -> float:
        return decode_f16(self)

    def is_nan(self) -> bool:
        return (self.bits & 0x7C00) == 0x7C00 and (self.bits & 0x03FF) != 0


def encode_f16(x: float) -> Binary16:
    """Round to binary16 (RNE, overflow to inf), NaN canonicalised (numerics.py:57-63)."""
    if math.isnan(x):
        return Binary16(NAN_BITS)
    with np.errstate(over="ignore"):
        h = np.float16(np.float64(x))
    return Binary16(int(h.view(np.uint16)))


def decode_f16(v: Binary16) -> float:
    return float(np.uint16(v.bits).view(np.float16))
