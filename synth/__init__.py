"""Seeded, counter-based synthetic input generators.

This module is the ONLY code shared between the CPU oracle (``oracle/``) and
the CUDA product path (``paper_2503_10725_b200``).  It holds none of the
Samoyeds method's arithmetic: it only turns (seed, flat index) into input
values.  The CUDA library carries a twin of the same generator
(``csrc/synth.cu``, exported as ``smy_synth_fill``) so that multi-GB weights can
be generated on the device; ``tests/test_gpu_parity.py::test_synth_twin_bit_exact``
pins the two bit-exactly.

Generator: a splitmix64-style finaliser over ``key(seed) + (i + 1) * PHI``.
Every distribution below is computed with exactly representable integer steps
followed by ONE fp32 multiply (round-to-nearest-even), so numpy and CUDA agree
bit for bit.  bf16 inputs are the fp32 value rounded to nearest-even bf16.

Input recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * weights   ~ U(-sqrt(3/k), sqrt(3/k)) (variance 1/k, as N(0,1/k)) -> bf16
  * activations, router logits ~ Irwin-Hall(4) scaled to unit variance
  * integer variant: values uniform in {lo..hi} (bit-exact SSMM checks)
Seeds: weights 1000 + 3e + {0 gate, 1 up, 2 down}; x 1; logits 2; skew 3.
"""
from __future__ import annotations

import numpy as np

PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

DIST_UNIFORM = 0   # (2u - 1) * scale, u = 24-bit uniform
DIST_NORMAL = 1    # (n1+n2+n3+n4 - 2^25) * scale, n_i = 24-bit uniforms
DIST_INT = 2       # lo + (h >> 32) % (hi - lo + 1)

SEED_X = 1
SEED_LOGITS = 2
SEED_SKEW = 3


def weight_seed(expert: int, which: int) -> int:
    """which: 0 = gate, 1 = up, 2 = down (SURVEY.md §8(d) seeds)."""
    return 1000 + 3 * expert + which


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def key(seed: int) -> np.uint64:
    return _mix(np.array([seed], dtype=np.uint64) * PHI + PHI)[0]


def hash64(seed: int, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(key(seed) + (idx + np.uint64(1)) * PHI)


def normal_scale(sigma: float) -> np.float32:
    """fp32 multiplier turning the integer Irwin-Hall(4) sum into std=sigma."""
    # Var(sum of 4 U(0,1)) = 1/3, the integer sum is in units of 2^-24.
    return np.float32(sigma * np.sqrt(3.0) / float(1 << 24))


def uniform_scale(half_width: float) -> np.float32:
    return np.float32(half_width / float(1 << 24))


def fill_f32(seed: int, idx: np.ndarray, dist: int, scale: float,
             lo: int = -2, hi: int = 2) -> np.ndarray:
    """Values at flat indices ``idx`` as float32 (bit-exact with the CUDA twin).

    ``scale`` is the fp32 multiplier (see normal_scale / uniform_scale); for
    DIST_INT it is ignored.
    """
    h = hash64(seed, idx)
    if dist == DIST_UNIFORM:
        n = (h >> np.uint64(40)).astype(np.int64)          # [0, 2^24)
        s = (2 * n - (1 << 24)).astype(np.float32)          # exact: |s| < 2^24
        return (s * np.float32(scale)).astype(np.float32)
    if dist == DIST_NORMAL:
        h2 = hash64(seed ^ 0x5DEECE66D, idx)
        n1 = (h >> np.uint64(40)).astype(np.int64)
        n2 = ((h >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.int64)
        n3 = (h2 >> np.uint64(40)).astype(np.int64)
        n4 = ((h2 >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.int64)
        s = (n1 + n2 + n3 + n4 - (1 << 25)).astype(np.float32)   # int -> f32 RNE
        return (s * np.float32(scale)).astype(np.float32)
    if dist == DIST_INT:
        span = np.uint64(hi - lo + 1)
        v = ((h >> np.uint64(32)) % span).astype(np.int64) + lo
        return v.astype(np.float32)
    raise ValueError(f"unknown dist {dist}")


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round to nearest even (input preparation)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = (u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ---------------------------------------------------------------- tensors

def weight_bf16(seed: int, rows: int, cols: int, row_idx=None, integer=False) -> np.ndarray:
    """bf16 bits of a [rows x cols] weight (or of the rows in ``row_idx``)."""
    r = np.arange(rows) if row_idx is None else np.asarray(row_idx)
    idx = (r.astype(np.uint64)[:, None] * np.uint64(cols)
           + np.arange(cols, dtype=np.uint64)[None, :])
    if integer:
        v = fill_f32(seed, idx, DIST_INT, 0.0)
    else:
        v = fill_f32(seed, idx, DIST_UNIFORM, uniform_scale(np.sqrt(3.0 / cols)))
    return f32_to_bf16_bits(v)


def activations_bf16(seed: int, rows: int, cols: int, row_idx=None, integer=False) -> np.ndarray:
    r = np.arange(rows) if row_idx is None else np.asarray(row_idx)
    idx = (r.astype(np.uint64)[:, None] * np.uint64(cols)
           + np.arange(cols, dtype=np.uint64)[None, :])
    if integer:
        v = fill_f32(seed, idx, DIST_INT, 0.0)
    else:
        v = fill_f32(seed, idx, DIST_NORMAL, normal_scale(1.0))
    return f32_to_bf16_bits(v)


def router_logits(seed: int, tokens: int, experts: int, skew: float = 0.0) -> np.ndarray:
    """fp32 [tokens x experts]; skew>0 adds a log-Zipf(s=skew) per-expert bias."""
    idx = np.arange(tokens * experts, dtype=np.uint64).reshape(tokens, experts)
    v = fill_f32(seed, idx, DIST_NORMAL, normal_scale(1.0))
    if skew:
        bias = (-skew * np.log(np.arange(1, experts + 1, dtype=np.float64))).astype(np.float32)
        v = (v + bias[None, :]).astype(np.float32)
    return v


def selection(seed: int, total: int, n_sel: int) -> np.ndarray:
    """n_sel distinct ascending ids in [0,total): the n_sel smallest hashes."""
    h = hash64(seed, np.arange(total, dtype=np.uint64))
    order = np.lexsort((np.arange(total), h))
    return np.sort(order[:n_sel]).astype(np.int32)
