"""Dual-side sparse SSMM reference -- oracle (TEST INFRASTRUCTURE).

The kernel scheme (Alg. 1) computes C = decode(W) x B[:, SEL]:
  "only len_d columns from matrix B are selected for computation, which are
   recorded in the selection array"
and is "mathematically equivalent with the original computation process"
(P:239).  So the oracle is that definition written out: decode the
weight to dense, gather the selected token rows, multiply in fp64 (library
matmul as one step).  Fused epilogues (§4.3 "Operator fusion"):
  * COMPACT          C stored for the selected tokens only (compressed
                     output layout)
  * SILU_MUL_COMPACT bf16( silu(C_gate) * C_up ) -- gate/up with the
                     activation fused (R11: SiLU gated MLP; R12: the
                     intermediate is stored as bf16, emulated with RNE)
  * SILU_MUL_INTERLEAVED  the same on one weight holding gate and up rows
                     interleaved in blocks of 16 compressed rows
                     (fmt.interleave_rows / gu_block, R20)
  * SCATTER_ADD      out[sel[t]] += scale[t] * C[t] -- "the weighted
                     accumulation ... is fused with matrix multiplication"

Layouts: x is [x_rows x k] bf16 bits, token-major ("the input x ...
row-major"); outputs are token-major [n_sel x m].
Error scale (north star): S[t, o] = sum_k |W[o,k] * x[t,k]|, used for the
per-element bound |err| <= 1e-2 * S.
"""
from __future__ import annotations

import numpy as np

from . import bf16
from .fmt import Encoded, dense_f64
from .fmt import deinterleave_rows as fmt_deinterleave


def _silu(h: np.ndarray) -> np.ndarray:
    return h / (1.0 + np.exp(-h))


def ssmm(enc: Encoded, x_bits: np.ndarray, sel: np.ndarray) -> np.ndarray:
    """C[t, o] = sum_k W[o, k] * x[sel[t], k]  in fp64; [len(sel) x rows]."""
    w = dense_f64(enc)
    xs = bf16.to_f64(np.asarray(x_bits)[np.asarray(sel, dtype=np.int64)])
    if xs.shape[0] == 0:
        return np.zeros((0, enc.rows))
    return xs @ w.T


def ssmm_abs(enc: Encoded, x_bits: np.ndarray, sel: np.ndarray) -> np.ndarray:
    """S[t, o] = sum_k |W[o,k] x[sel[t],k]| (error scale)."""
    w = np.abs(dense_f64(enc))
    xs = np.abs(bf16.to_f64(np.asarray(x_bits)[np.asarray(sel, dtype=np.int64)]))
    if xs.shape[0] == 0:
        return np.zeros((0, enc.rows))
    return xs @ w.T


def silu_mul_bf16(c_gate: np.ndarray, c_up: np.ndarray) -> np.ndarray:
    """bf16 bits of silu(C_gate) * C_up, RNE from fp64 (R12)."""
    return bf16.from_f64(_silu(c_gate) * c_up)


def silu_mul_interleaved_bf16(c_gu: np.ndarray) -> np.ndarray:
    """SILU_MUL_INTERLEAVED epilogue: C_gu = C of the interleaved gate/up
    weight (fmt.interleave_rows, reading R20) [n x 2f]; the output column o < f
    is bf16(silu(C_gate[:, o]) * C_up[:, o]) with the gate/up columns recovered
    by the inverse relabeling."""
    g, u = fmt_deinterleave(np.asarray(c_gu).T)
    return silu_mul_bf16(g.T, u.T)


def scatter_add(out: np.ndarray, c: np.ndarray, sel_out: np.ndarray, scale=None) -> np.ndarray:
    """out[sel_out[t]] += scale[t] * c[t]  (fp64, returns a new array)."""
    out = np.array(out, dtype=np.float64, copy=True)
    s = np.ones(len(sel_out)) if scale is None else np.asarray(scale, dtype=np.float64)
    for t, dst in enumerate(np.asarray(sel_out, dtype=np.int64)):
        out[dst] += s[t] * c[t]
    return out


def masked_dense_reference(w_dense_bits_pruned: np.ndarray, x_bits: np.ndarray,
                           sel: np.ndarray) -> np.ndarray:
    """Brute-force check path: element-by-element triple loop over the pruned
    dense weight (no encoding involved).  Tiny inputs only."""
    w = bf16.to_f64(w_dense_bits_pruned)
    x = bf16.to_f64(x_bits)
    out = np.zeros((len(sel), w.shape[0]))
    for t, tok in enumerate(sel):
        for o in range(w.shape[0]):
            acc = 0.0
            for k in range(w.shape[1]):
                if w[o, k] != 0.0:
                    acc += w[o, k] * x[tok, k]
            out[t, o] = acc
    return out


def rel_fro(err: np.ndarray, ref: np.ndarray) -> float:
    num = float(np.sqrt(np.sum(np.square(err, dtype=np.float64))))
    den = float(np.sqrt(np.sum(np.square(ref, dtype=np.float64))))
    return num / den if den else num
