"""Device images of an encoded weight -- oracle (TEST INFRASTRUCTURE).

The paper packs A, B and the metadata for the Ampere/Ada ``mma.sp.m16n8k32``
register fragments (§4.4).  On sm_100a the same three streams feed
``tcgen05.mma.sp`` instead, so the packing targets its operand layouts.  This
module writes those layouts out from their documentation (DESIGN.md §HBM
layout), independently of the CUDA packer, so the GPU packer can be checked
bit-exactly and the end-to-end SSMM parity tests check that the hardware reads
them the way they are documented.

One weight image = [m_tiles][k_stages] blocks of IMG_BLOCK bytes:

  block = | A  16384 B | E  2048 B | planes 64*P B | zero pad to IMG_BLOCK |

  m_tile  : 128 compressed rows (TMEM lanes); rows >= R are zero
  k_stage : 4 "virtual K-blocks" of 32 logical K each (one tcgen05.mma.sp
            bf16 covers K=32).  For V=32 a virtual block is a real K-block.
            For V=16 (rep=2) each real 32-block is issued twice: virtual block
            (j, h) keeps only the 16-wide sub-block h, the other half's value
            slots are zero (D4).

  A: the 128 x 64 bf16 (128 B per row) smem image of the stage's compressed
     values, K-major, 128-byte swizzle: row r, 16-byte chunk c lives at
     (r//8)*1024 + (r%8)*128 + ((c ^ (r%8)) * 16).
  E: the TMEM image of the 2:4 metadata, 128 lanes x 4 columns x 32 bit,
     lane-major (lane l at byte 16*l, column kb at +4*kb).  Lane l carries
     rows r_lo = (l%8) + 16*(l//16) and r_hi = r_lo + 8 of K-half
     k1 = (l//8)%2; bits [0,16) = row r_lo, bits [16,32) = row r_hi; inside a
     16-bit half, nibble q holds the code pair of 4-group 4*k1+q as
     p0 | p1 << 2.
  planes: for each virtual K-block kb and plane b < P = ceil(log2 M) (P = 0
     when N == M), 128 bits: bit l = bit b of idx[row l].  Word w of a plane
     holds lanes 32w..32w+31.
"""
from __future__ import annotations

import math

import numpy as np

from .fmt import Encoded, SparseFormat

TILE_M = 128
STAGE_VK = 128            # virtual logical K per stage (4 x K=32)
A_BYTES = 16384
E_BYTES = 2048


def n_planes(fmt: SparseFormat) -> int:
    return 0 if fmt.n == fmt.m else max(1, math.ceil(math.log2(fmt.m)))


def rep(fmt: SparseFormat) -> int:
    if 32 % fmt.v and fmt.v % 32:
        raise ValueError("V must divide 32 or be a multiple of 32")
    return max(1, 32 // fmt.v)


def img_block(fmt: SparseFormat) -> int:
    b = A_BYTES + E_BYTES + 64 * n_planes(fmt)
    return (b + 255) // 256 * 256


def geometry(rows: int, cols: int, fmt: SparseFormat) -> dict:
    R = fmt.comp_rows(rows)
    vk = cols * rep(fmt)
    if vk % STAGE_VK:
        raise ValueError("K * rep must be a multiple of 128")
    return dict(R=R, m_tiles=(R + TILE_M - 1) // TILE_M, k_stages=vk // STAGE_VK,
                planes=n_planes(fmt), block=img_block(fmt), rep=rep(fmt))


def _virtual(enc: Encoded):
    """Per virtual K-block: values [R, nvb, 16] bits, codes [R, nvb, 8, 2],
    routing idx [R, nvb]."""
    fmt = enc.fmt
    R = fmt.comp_rows(enc.rows)
    rp = rep(fmt)
    nreal = enc.cols // 32                       # real 32-wide blocks
    val = enc.values.reshape(R, nreal, 8, 2)     # chunk q of the 32-block: slots 2q, 2q+1
    cod = enc.codes.reshape(R, nreal, 8, 2)
    nvb = nreal * rp
    v = np.zeros((R, nvb, 8, 2), dtype=np.uint16)
    c = np.zeros((R, nvb, 8, 2), dtype=np.uint8)
    c[..., 1] = 1                                # dead chunks: valid pair (0,1), value 0
    ridx = np.zeros((R, nvb), dtype=np.int64)
    for j in range(nreal):
        for h in range(rp):
            vb = j * rp + h
            live = slice(0, 8) if rp == 1 else slice(4 * h, 4 * h + 4)
            v[:, vb, live] = val[:, j, live]
            c[:, vb, live] = cod[:, j, live]
            vblock = (j * 32 + (live.start * 4)) // fmt.v     # V-block of the live chunks
            ridx[:, vb] = enc.idx[:, vblock]
    return v.reshape(R, nvb, 16), c, ridx


def a_image(enc: Encoded) -> np.ndarray:
    """uint8 [m_tiles, k_stages, 16384]."""
    g = geometry(enc.rows, enc.cols, enc.fmt)
    v, _, _ = _virtual(enc)
    R, mt, ks = g["R"], g["m_tiles"], g["k_stages"]
    img = np.zeros((mt, ks, A_BYTES), dtype=np.uint8)
    vals = np.zeros((mt * TILE_M, ks * 64), dtype=np.uint16)
    vals[:R] = v.reshape(R, -1)
    for t in range(mt):
        for s in range(ks):
            blk = vals[t * TILE_M:(t + 1) * TILE_M, s * 64:(s + 1) * 64]    # 128 x 64
            for r in range(TILE_M):
                for ch in range(8):
                    off = (r // 8) * 1024 + (r % 8) * 128 + ((ch ^ (r % 8)) * 16)
                    img[t, s, off:off + 16] = blk[r, ch * 8:(ch + 1) * 8].view(np.uint8)
    return img


def e_image(enc: Encoded) -> np.ndarray:
    """uint8 [m_tiles, k_stages, 2048]."""
    g = geometry(enc.rows, enc.cols, enc.fmt)
    _, c, _ = _virtual(enc)                      # [R, nvb, 8, 2]
    R, mt, ks = g["R"], g["m_tiles"], g["k_stages"]
    nib = np.zeros((mt * TILE_M, ks * 4, 8), dtype=np.uint32)
    nib[:, :, :] = 0x4                           # padding rows: pair (0,1)
    nib[:R] = (c[..., 0].astype(np.uint32) | (c[..., 1].astype(np.uint32) << 2))
    img = np.zeros((mt, ks, 128, 4), dtype=np.uint32)
    for t in range(mt):
        for s in range(ks):
            for lane in range(128):
                r_lo = (lane % 8) + 16 * (lane // 16)
                r_hi = r_lo + 8
                k1 = (lane // 8) % 2
                for kb in range(4):
                    word = 0
                    for q in range(4):
                        word |= int(nib[t * TILE_M + r_lo, s * 4 + kb, 4 * k1 + q]) << (4 * q)
                        word |= int(nib[t * TILE_M + r_hi, s * 4 + kb, 4 * k1 + q]) << (16 + 4 * q)
                    img[t, s, lane, kb] = word
    return img.view(np.uint8).reshape(mt, ks, E_BYTES)


def planes(enc: Encoded) -> np.ndarray:
    """uint8 [m_tiles, k_stages, 64*P]."""
    g = geometry(enc.rows, enc.cols, enc.fmt)
    P = g["planes"]
    _, _, ridx = _virtual(enc)
    R, mt, ks = g["R"], g["m_tiles"], g["k_stages"]
    full = np.zeros((mt * TILE_M, ks * 4), dtype=np.int64)
    full[:R] = ridx
    out = np.zeros((mt, ks, 4, max(P, 1), 4), dtype=np.uint32)
    for t in range(mt):
        for s in range(ks):
            for kb in range(4):
                for b in range(P):
                    for lane in range(128):
                        if (full[t * TILE_M + lane, s * 4 + kb] >> b) & 1:
                            out[t, s, kb, b, lane // 32] |= np.uint32(1 << (lane % 32))
    if P == 0:
        return np.zeros((mt, ks, 0), dtype=np.uint8)
    return np.ascontiguousarray(out[:, :, :, :P, :]).view(np.uint8).reshape(mt, ks, 64 * P)


def weight_image(enc: Encoded) -> np.ndarray:
    """uint8 [m_tiles * k_stages * IMG_BLOCK]: the whole device image."""
    g = geometry(enc.rows, enc.cols, enc.fmt)
    a, e, p = a_image(enc), e_image(enc), planes(enc)
    blk = np.zeros((g["m_tiles"], g["k_stages"], g["block"]), dtype=np.uint8)
    blk[:, :, :A_BYTES] = a
    blk[:, :, A_BYTES:A_BYTES + E_BYTES] = e
    if g["planes"]:
        blk[:, :, A_BYTES + E_BYTES:A_BYTES + E_BYTES + 64 * g["planes"]] = p
    return blk.reshape(-1)
