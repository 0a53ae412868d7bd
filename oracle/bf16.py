"""bf16 helpers for the oracle (exact, bit level).

bf16 is the operand type of the paper's kernels ("metadata in bfloat type",
P:352 §4.4).  bf16 -> fp64 is exact (u16 << 16 reinterpreted as fp32).
fp64 -> bf16 rounds to nearest-even DIRECTLY from fp64 (no double rounding
through fp32); R12.
"""
from __future__ import annotations

import numpy as np


def to_f64(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def _trunc_bits(ax: np.ndarray) -> np.ndarray:
    """Bits of the largest bf16 magnitude <= ax (ax >= 0, finite, fp64)."""
    f = ax.astype(np.float32)                       # nearest fp32
    fb = f.view(np.uint32)
    up = f.astype(np.float64) > ax                  # rounded up -> step down one ulp
    fb = np.where(up & (fb > 0), fb - 1, fb).astype(np.uint32)
    return (fb >> np.uint32(16)).astype(np.uint16)  # chop to bf16 (toward zero)


def from_f64(x: np.ndarray) -> np.ndarray:
    """Round fp64 to the nearest bf16, ties to even; returns uint16 bits."""
    x = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite value in bf16 rounding")
    ax = np.abs(x)
    lo_bits = _trunc_bits(ax)
    hi_bits = (lo_bits.astype(np.uint32) + 1).astype(np.uint16)
    d_lo = ax - to_f64(lo_bits)
    d_hi = to_f64(hi_bits) - ax
    pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & ((lo_bits & 1) == 1))
    mag = np.where(pick_hi, hi_bits, lo_bits).astype(np.uint16)
    sign = np.signbit(x).astype(np.uint16) << np.uint16(15)
    return (mag | sign).astype(np.uint16)


def round_f64(x: np.ndarray) -> np.ndarray:
    """fp64 value of the bf16 nearest to x."""
    return to_f64(from_f64(x))
