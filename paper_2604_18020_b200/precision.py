"""Working-precision policies (reference precision.py:25-99).

The B200 hot path computes in FP32 or FP64.  The reference's emulated
bfloat16 ("bf16": FP32 storage, every term bf16-rounded) is served by the
general-connectivity bf16 kernels (csrc/tf_bf16.cu) exactly as the reference
defines it -- the documented negative result (PAPER.md:1522-1552,
DESIGN.md §9); the structured production kernels and tensor cores are never
used for it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

EPS_FP64 = 2.0**-53
EPS_FP32 = 2.0**-24
EPS_BF16 = 2.0**-8
BF16_MAX = float(2.0**127 * (255.0 / 128.0))


@dataclass(frozen=True)
class Precision:
    tag: str
    unit_roundoff: float

    @property
    def dtype(self):
        return np.float64 if self.tag == "fp64" else np.float32

    @property
    def scalar_bytes(self) -> int:
        return 8 if self.tag == "fp64" else 4

    @property
    def quantized(self) -> bool:
        return self.tag == "bf16"


FP64 = Precision("fp64", EPS_FP64)
FP32 = Precision("fp32", EPS_FP32)
BF16 = Precision("bf16", EPS_BF16)
_BY_TAG = {p.tag: p for p in (FP64, FP32, BF16)}


def get_precision(tag: str) -> Precision:
    if tag not in _BY_TAG:
        raise ValueError(f"unknown precision tag {tag!r}, expected fp64|fp32|bf16")
    return _BY_TAG[tag]


def round_to_bf16(x):
    """Round-to-nearest-even onto the bfloat16 grid, returned as float32.

    NaNs are quieted, infinities and signed zeros pass through, overflow goes
    to infinity (reference precision.py:65-85 semantics).
    """
    a = np.asarray(x, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    special = (bits & 0x7F800000) == 0x7F800000
    lsb = (bits >> 16) & 1
    rounded = ((bits + 0x7FFF + lsb) >> 16) << 16
    trunc = (bits >> 16) << 16
    is_nan = special & ((bits & 0x007FFFFF) != 0)
    out = np.where(special, np.where(is_nan, trunc | 0x00400000, trunc), rounded)
    res = (out & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    if np.ndim(x) == 0:
        return np.float32(res.reshape(()))
    return res


def quantize(v, precision: Precision):
    if precision.tag == "fp64":
        return np.asarray(v, dtype=np.float64)
    if precision.tag == "fp32":
        return np.asarray(v, dtype=np.float32)
    return round_to_bf16(np.asarray(v, dtype=np.float32))
