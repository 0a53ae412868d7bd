"""Samoyeds dual-side sparse weight format -- oracle (TEST INFRASTRUCTURE).

Paper: §4.1, Fig. 7 "Samoyeds Dual-side Sparse Data Format".

  "The original weight data is segmented into structured sparse blocks of size
   M x V. Each vector within a block, termed as a Sub-Row, contains multiple
   SpTC units. Within each block, only N Sub-Rows are retained ... The SpTC
   units within the selected Sub-Row are further pruned to conform to the
   sparse pattern supported by the hardware."
  "the original weight is encoded into three components: data, indices, and
   metadata ... data m/M x k/2 ... indices m/M x k/V ... metadata m/M x k/2
   ... encoded into 2-bits"

Readings: R1 shapes use rows*N/M (P:237 is only right for N=1);
R2 sub-row = 1 x V along K, block = M output rows x V reduction columns;
R3 one 2-bit code per stored value; R4 magnitude selection (fp32 sequential
L1 for sub-rows, |w| for elements, ties -> lower index); R5 fewer than N
non-zero sub-rows -> fill with the lowest-index unused sub-rows; R6 fewer than
2 non-zeros in a 4-group -> pad with the smallest unused positions; R7 codes
packed LSB-first 4 per byte.

Weights are uint16 bf16 bit patterns, shape [rows x cols] = [out x in]
(PyTorch layout, the paper's W^T after the offline transposition).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class FormatError(ValueError):
    pass


class ShapeError(FormatError):
    pass


class PatternError(FormatError):
    pass


class CorruptFormat(FormatError):
    pass


@dataclass(frozen=True)
class SparseFormat:
    """(N, M, V): keep N of every M sub-rows of length V, then 2:4 inside."""
    n: int
    m: int
    v: int

    def __post_init__(self):
        if not (1 <= self.n <= self.m):
            raise ShapeError(f"need 1 <= N <= M, got {self}")
        if self.v <= 0 or self.v % 4:
            raise ShapeError(f"V must be a positive multiple of 4, got {self}")

    @property
    def density(self) -> float:
        """Fraction of weights kept: (N/M) * (2/4)."""
        return self.n / self.m * 0.5

    def comp_rows(self, rows: int) -> int:
        return rows * self.n // self.m


# Table 4 / P:589 configurations
TABLE4 = (SparseFormat(1, 2, 16), SparseFormat(1, 2, 32),
          SparseFormat(4, 8, 32), SparseFormat(8, 16, 32))


def check_shape(rows: int, cols: int, fmt: SparseFormat) -> None:
    if rows % fmt.m or cols % fmt.v:
        raise ShapeError(f"[{rows}x{cols}] not divisible by (M={fmt.m}, V={fmt.v})")


def _nonzero(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16) & np.uint16(0x7FFF)) != 0


def _abs_f32(bits: np.ndarray) -> np.ndarray:
    b = (np.asarray(bits, dtype=np.uint16) & np.uint16(0x7FFF)).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32)


# ------------------------------------------------------------------ prune (R4)

def subrow_scores(w_bits: np.ndarray, fmt: SparseFormat) -> np.ndarray:
    """L1 score of every sub-row, fp32, summed sequentially in ascending column
    order (R4).  Returns [rows, cols/V]."""
    rows, cols = w_bits.shape
    check_shape(rows, cols, fmt)
    a = _abs_f32(w_bits).reshape(rows, cols // fmt.v, fmt.v)
    acc = np.zeros((rows, cols // fmt.v), dtype=np.float32)
    for c in range(fmt.v):                       # sequential fp32 sum, no reassociation
        acc = (acc + a[:, :, c]).astype(np.float32)
    return acc


def prune(w_bits: np.ndarray, fmt: SparseFormat) -> np.ndarray:
    """Magnitude pruning to the (N,M,V)+2:4 pattern (R4).

    In every M x V block keep the N sub-rows with the highest L1 score (ties ->
    lower row); inside each kept sub-row keep, per aligned 4-group, the two
    largest |w| (ties -> lower position).  Everything else becomes +0.
    """
    w_bits = np.asarray(w_bits, dtype=np.uint16)
    rows, cols = w_bits.shape
    check_shape(rows, cols, fmt)
    G, M, J, V = rows // fmt.m, fmt.m, cols // fmt.v, fmt.v
    score = subrow_scores(w_bits, fmt).reshape(G, M, J)
    # rank of each sub-row inside its block: #rows that beat it
    s_i = score[:, :, None, :]                   # candidate
    s_o = score[:, None, :, :]                   # others
    r_i = np.arange(M)[None, :, None, None]
    r_o = np.arange(M)[None, None, :, None]
    beats = (s_o > s_i) | ((s_o == s_i) & (r_o < r_i))
    keep_row = beats.sum(axis=2) < fmt.n         # [G, M, J]
    a = _abs_f32(w_bits).reshape(G, M, J, V // 4, 4)
    a_i = a[..., :, None]
    a_o = a[..., None, :]
    p_i = np.arange(4)[:, None]
    p_o = np.arange(4)[None, :]
    beats_e = (a_o > a_i) | ((a_o == a_i) & (p_o < p_i))
    keep_el = beats_e.sum(axis=-1) < 2           # [G, M, J, V/4, 4]
    keep = keep_el & keep_row[:, :, :, None, None]
    out = np.where(keep, w_bits.reshape(G, M, J, V // 4, 4), np.uint16(0))
    return out.reshape(rows, cols).astype(np.uint16)


# ------------------------------------------------------------ encode / decode

@dataclass
class Encoded:
    """Canonical encoding: values [R x cols/2] bf16 bits, codes
    [R x cols/2] in 0..3, idx [R x cols/V] in 0..M-1, R = rows*N/M (R1)."""
    rows: int
    cols: int
    fmt: SparseFormat
    values: np.ndarray
    codes: np.ndarray
    idx: np.ndarray


def encode(w_bits: np.ndarray, fmt: SparseFormat) -> Encoded:
    """Encode a pattern-conforming weight (R5, R6)."""
    w_bits = np.asarray(w_bits, dtype=np.uint16)
    rows, cols = w_bits.shape
    check_shape(rows, cols, fmt)
    G, M, N, J, V = rows // fmt.m, fmt.m, fmt.n, cols // fmt.v, fmt.v
    blk = w_bits.reshape(G, M, J, V)
    nzrow = _nonzero(blk).any(axis=3)                          # [G, M, J]
    if (nzrow.sum(axis=1) > N).any():
        raise PatternError("a block has more than N non-zero sub-rows")
    # non-zero rows first in index order, then unused rows in index order (R5)
    key = (~nzrow).astype(np.int64) * M + np.arange(M)[None, :, None]
    pick = np.sort(np.argsort(key, axis=1, kind="stable")[:, :N, :], axis=1)   # [G, N, J]
    sub = np.take_along_axis(blk, pick[..., None], axis=1)     # [G, N, J, V]
    grp = sub.reshape(G, N, J, V // 4, 4)
    nz = _nonzero(grp)
    if (nz.sum(axis=-1) > 2).any():
        raise PatternError("a 4-group has more than 2 non-zeros")
    key4 = (~nz).astype(np.int64) * 4 + np.arange(4)
    pos = np.sort(np.argsort(key4, axis=-1, kind="stable")[..., :2], axis=-1)  # [G,N,J,V/4,2]
    vals = np.take_along_axis(grp, pos, axis=-1)
    R = G * N
    values = vals.reshape(R, J * (V // 2)).astype(np.uint16)
    codes = pos.reshape(R, J * (V // 2)).astype(np.uint8)
    idx = pick.reshape(R, J).astype(np.uint8)
    return Encoded(rows, cols, fmt, values, codes, idx)


def validate(enc: Encoded) -> list:
    """Invariant violations of an encoding; empty list if valid."""
    out = []
    fmt = enc.fmt
    R = fmt.comp_rows(enc.rows)
    J = enc.cols // fmt.v
    if enc.values.shape != (R, enc.cols // 2) or enc.codes.shape != (R, enc.cols // 2) \
            or enc.idx.shape != (R, J):
        return [("shape", None)]
    idx = enc.idx.astype(np.int64).reshape(R // fmt.n, fmt.n, J)
    for g, i, j in zip(*np.nonzero(idx >= fmt.m)):
        out.append(("index_out_of_range", (int(g * fmt.n + i), int(j))))
    if fmt.n > 1:
        bad = np.diff(idx, axis=1) <= 0
        for g, i, j in zip(*np.nonzero(bad)):
            out.append(("index_not_increasing", (int(g), int(j))))
    c = enc.codes.astype(np.int64).reshape(R, enc.cols // 4, 2)
    for r, q in zip(*np.nonzero((c[..., 0] >= c[..., 1]) | (c[..., 1] > 3))):
        out.append(("metadata_not_increasing", (int(r), int(q))))
    return out


def decode(enc: Encoded) -> np.ndarray:
    """Inverse of encode (survey §8(c) step 4): scatter every stored
    value to W[g*M + idx, j*V + 4q + code]; everything else 0."""
    bad = validate(enc)
    if bad:
        raise CorruptFormat(f"invalid encoding: {bad[:4]}")
    fmt = enc.fmt
    R = fmt.comp_rows(enc.rows)
    J, V = enc.cols // fmt.v, fmt.v
    w = np.zeros((enc.rows, enc.cols), dtype=np.uint16)
    written = np.zeros((enc.rows, enc.cols), dtype=bool)
    r = np.arange(R)[:, None]
    c = np.arange(enc.cols // 2)[None, :]
    j = (2 * c) // V                            # K-block of stored slot c
    q = (c % (V // 2)) // 2                     # 4-group inside the block
    row = (r // fmt.n) * fmt.m + enc.idx[r, j].astype(np.int64)
    col = j * V + 4 * q + enc.codes.astype(np.int64)
    if written[row, col].any() or len(np.unique(row * enc.cols + col)) != row.size:
        raise CorruptFormat("two stored values map to one position")
    w[row, col] = enc.values
    return w


def dense_f64(enc: Encoded) -> np.ndarray:
    from .bf16 import to_f64
    return to_f64(decode(enc))


# -------------------------------------------------------- canonical packing (R7)

def pack_codes(codes: np.ndarray) -> np.ndarray:
    """2-bit codes -> bytes, 4 per byte, code c at bits 2*(c mod 4) (R7)."""
    R, C = codes.shape
    assert C % 4 == 0
    c = codes.astype(np.uint8).reshape(R, C // 4, 4)
    return (c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)).astype(np.uint8)


def unpack_codes(packed: np.ndarray) -> np.ndarray:
    R, B = packed.shape
    p = packed.astype(np.uint8)
    return np.stack([(p >> s) & 3 for s in (0, 2, 4, 6)], axis=-1).reshape(R, B * 4).astype(np.uint8)


# ------------------------------------------------ paper Fig. 10 panel packing

def pack_panel(meta16: np.ndarray) -> np.ndarray:
    """§4.4: element [r, c] of a 16x16 2-bit panel moves to
    [r % 8 * 2 + c / 8, c % 8 + r / 8 * 8].  Reference transform only: the
    B200 kernel uses the tcgen05 E layout (devlayout.py) instead."""
    meta16 = np.asarray(meta16)
    if meta16.shape != (16, 16):
        raise ShapeError("panel must be 16x16")
    out = np.empty_like(meta16)
    for r in range(16):
        for c in range(16):
            out[r % 8 * 2 + c // 8, c % 8 + r // 8 * 8] = meta16[r, c]
    return out


def unpack_panel(packed: np.ndarray) -> np.ndarray:
    packed = np.asarray(packed)
    if packed.shape != (16, 16):
        raise ShapeError("panel must be 16x16")
    out = np.empty_like(packed)
    for r in range(16):
        for c in range(16):
            out[r, c] = packed[r % 8 * 2 + c // 8, c % 8 + r // 8 * 8]
    return out


# --------------------------------------------------------------- byte sizes

def canonical_bytes(rows: int, cols: int, fmt: SparseFormat, elem_bytes: int = 2) -> dict:
    """Closed-form sizes of the canonical encoding."""
    R = fmt.comp_rows(rows)
    return {
        "dense": rows * cols * elem_bytes,
        "values": R * (cols // 2) * elem_bytes,
        "codes": R * (cols // 2) * 2 // 8,
        "indices": R * (cols // fmt.v),
    }


# ------------------------------------------- interleaved gate/up (reading R20)

GU_BLOCK = 32    # output rows per interleave block for N/M = 1/2 formats
GU_CBLOCK = 16   # compressed rows per interleave block (every format, R20)


def gu_block(fmt: "SparseFormat") -> int:
    """Output rows per interleave block of a format: 16 compressed rows, i.e. 32
    output rows for N/M = 1/2 and 16 for N = M (R20)."""
    return GU_CBLOCK * fmt.m // fmt.n


def interleave_rows(w_gate: np.ndarray, w_up: np.ndarray, block: int = GU_BLOCK) -> np.ndarray:
    """Dense [2f x d] gate/up weight with the two projections interleaved in
    blocks of `block` output rows: rows [2b*block, (2b+1)*block) are gate rows
    [b*block, (b+1)*block) and the next `block` rows are the same up rows.

    The paper fuses the activation with "its precedent operator" but
    does not fix how gate and up share a kernel; this row relabeling (R20)
    puts the gate and up rows of the same 32 outputs into one 32-lane slice of
    a 128-lane tile (gate in lanes 0-15, up in 16-31 for N/M = 1/2)."""
    w_gate, w_up = np.asarray(w_gate), np.asarray(w_up)
    if w_gate.shape != w_up.shape or w_gate.shape[0] % block:
        raise ShapeError("gate/up must have equal shapes with rows % block == 0")
    f, d = w_gate.shape
    out = np.empty((2 * f, d), dtype=w_gate.dtype)
    for b in range(f // block):
        out[2 * b * block:(2 * b + 1) * block] = w_gate[b * block:(b + 1) * block]
        out[(2 * b + 1) * block:(2 * b + 2) * block] = w_up[b * block:(b + 1) * block]
    return out


def deinterleave_rows(w_gu: np.ndarray, block: int = GU_BLOCK):
    """Inverse of interleave_rows on the row axis: returns (gate, up).  Works
    on any array whose axis 0 is the interleaved row index."""
    w_gu = np.asarray(w_gu)
    nb = w_gu.shape[0] // (2 * block)
    gate = np.concatenate([w_gu[2 * b * block:(2 * b + 1) * block] for b in range(nb)])
    up = np.concatenate([w_gu[(2 * b + 1) * block:(2 * b + 2) * block] for b in range(nb)])
    return gate, up


def interleave_gate_up(eg: Encoded, eu: Encoded, block: int = None) -> Encoded:
    """Canonical encoding of interleave_rows(gate, up) built from the two
    encodings: a block of `block` output rows is block*N/M compressed rows
    (R1), so the relabeling moves whole compressed rows of values, codes and
    indices (no re-encoding)."""
    if block is None:
        block = gu_block(eg.fmt)
    if eg.fmt != eu.fmt or (eg.rows, eg.cols) != (eu.rows, eu.cols) or eg.rows % block:
        raise ShapeError("gate/up encodings must match and rows % block == 0")
    cb = eg.fmt.comp_rows(block)
    out = {}
    for name in ("values", "codes", "idx"):
        a, b = getattr(eg, name), getattr(eu, name)
        out[name] = interleave_rows(a, b, cb)
    return Encoded(2 * eg.rows, eg.cols, eg.fmt, out["values"], out["codes"], out["idx"])
