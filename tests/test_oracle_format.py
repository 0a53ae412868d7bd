"""Pins for oracle/fmt.py and oracle/bf16.py against the paper, SPEC goldens,
closed forms and brute force (CPU only)."""
import itertools
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import bf16, fmt as F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bits(a):
    return synth.f32_to_bf16_bits(np.asarray(a, dtype=np.float32))


# ---------------------------------------------------------------- bf16

def test_bf16_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32),
                        np.float32([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3e-39, -65504.0])])
    # halfway cases: exact ties between two bf16 neighbours
    base = bits(rng.standard_normal(2000)).astype(np.uint32) << 16
    ties = (base | 0x8000).view(np.float32)
    x = np.concatenate([x, ties])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = bf16.from_f64(x.astype(np.float64))
    assert np.array_equal(got, ref)
    assert np.array_equal(bf16.to_f64(got).astype(np.float32).view(np.uint32) >> 16, ref)


def test_bf16_direct_from_f64_no_double_rounding():
    # 1 + 2^-8 + 2^-30: fp32 would round to 1+2^-8 (a tie) then bf16 ties-to-even
    # gives 1.0; the exact value is above the tie, so the answer is 1 + 2^-7.
    x = np.array([1.0 + 2.0 ** -8 + 2.0 ** -30])
    assert bf16.to_f64(bf16.from_f64(x))[0] == 1.0 + 2.0 ** -7


# ---------------------------------------------------------------- prune

def test_prune_golden_tie():
    g = GOLD["prune_tie_124"]
    out = F.prune(bits(g["w"]), F.SparseFormat(*g["fmt"]))
    assert np.array_equal(bf16.to_f64(out), np.array(g["pruned"], dtype=np.float64))


def _brute_prune(w, fmt):
    """Brute force: enumerate the sub-row choice per block (max exact L1, ties
    lower row) and the pair per 4-group (max exact |a|+|b|, ties
    lexicographically smallest pair)."""
    rows, cols = w.shape
    out = np.zeros_like(w)
    for g in range(rows // fmt.m):
        for j in range(cols // fmt.v):
            blk = w[g * fmt.m:(g + 1) * fmt.m, j * fmt.v:(j + 1) * fmt.v]
            best = None
            for combo in itertools.combinations(range(fmt.m), fmt.n):
                s = [sum(abs(int(x)) for x in blk[r]) for r in combo]
                key = (tuple(sorted(s, reverse=True)), tuple(-r for r in combo))
                # compare by: each kept row must dominate every dropped row
                ok = all(sum(abs(int(x)) for x in blk[r]) > sum(abs(int(x)) for x in blk[d])
                         or (sum(abs(int(x)) for x in blk[r]) == sum(abs(int(x)) for x in blk[d]) and r < d)
                         for r in combo for d in range(fmt.m) if d not in combo)
                if ok:
                    best = combo
            for r in best:
                for q in range(fmt.v // 4):
                    grp = blk[r, 4 * q:4 * q + 4]
                    pairs = sorted(itertools.combinations(range(4), 2),
                                   key=lambda p: (-(abs(int(grp[p[0]])) + abs(int(grp[p[1]]))), p))
                    for p in pairs[0]:
                        out[g * fmt.m + r, j * fmt.v + 4 * q + p] = grp[p]
    return out


@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 4), F.SparseFormat(2, 4, 8), F.SparseFormat(1, 4, 4)])
def test_prune_brute_force_small_integers(fmt):
    """S:480 acceptance: exhaustive small instances against brute force, many ties."""
    rng = np.random.default_rng(1)
    shape = (4, 8) if fmt.m <= 2 else (8, 16)
    for _ in range(300):
        w = rng.integers(-3, 4, size=shape)
        got = bf16.to_f64(F.prune(bits(w), fmt))
        assert np.array_equal(got, _brute_prune(w, fmt).astype(np.float64)), w


@pytest.mark.parametrize("fmt", F.TABLE4)
def test_prune_properties(fmt):
    rng = np.random.default_rng(2)
    w = bits(rng.standard_normal((64, 128)))
    p = F.prune(w, fmt)
    assert np.array_equal(F.prune(p, fmt), p)                       # idempotent
    sc = bits(bf16.to_f64(w) * 4.0)                                 # exact power-of-two scaling
    assert np.array_equal(F.prune(sc, fmt) != 0, p != 0)            # scale invariance
    kept = np.count_nonzero(bf16.to_f64(p))
    assert kept == 64 * 128 * fmt.density                           # dense random: exactly N/M * 1/2
    F.encode(p, fmt)                                                # pattern valid


def test_subrow_score_is_sequential_fp32():
    # 2^24 + 1 + 1 ... : pairwise summation would differ from sequential
    row = np.float32([2.0 ** 24, 1.0, 1.0, 1.0])
    s = F.subrow_scores(bits(row)[None, :], F.SparseFormat(1, 1, 4))
    acc = np.float32(0)
    for v in bf16.to_f64(bits(row)).astype(np.float32):
        acc = np.float32(acc + v)
    assert s[0, 0] == acc == np.float32(2.0 ** 24)


# ---------------------------------------------------------- encode / decode

def test_encode_golden():
    g = GOLD["encode_124"]
    e = F.encode(bits(g["w"]), F.SparseFormat(*g["fmt"]))
    assert np.array_equal(bf16.to_f64(e.values), np.array(g["data"], dtype=np.float64))
    assert e.idx.tolist() == g["indices"]
    assert e.codes.tolist() == g["codes"]
    assert np.array_equal(F.decode(e), bits(g["w"]))


def test_encode_shapes_golden():
    g = GOLD["encode_shapes_1408x2048_1_2_16"]
    fmt = F.SparseFormat(*g["fmt"])
    w = F.prune(synth.weight_bf16(7, g["rows"], g["cols"]), fmt)
    e = F.encode(w, fmt)
    assert list(e.values.shape) == g["data"]
    assert list(e.idx.shape) == g["indices"]
    assert list(e.codes.shape) == g["metadata"]


@pytest.mark.parametrize("fmt", F.TABLE4 + (F.SparseFormat(2, 2, 32), F.SparseFormat(1, 1, 32),
                                            F.SparseFormat(2, 4, 8)))
def test_roundtrip(fmt):
    rng = np.random.default_rng(3)
    for _ in range(20):
        rows = fmt.m * int(rng.integers(1, 5))
        cols = fmt.v * int(rng.integers(1, 5)) * (32 // fmt.v if fmt.v < 32 else 1)
        w = bits(rng.standard_normal((rows, cols)) * (rng.random((rows, cols)) > 0.3))
        p = F.prune(w, fmt)
        e = F.encode(p, fmt)
        assert F.validate(e) == []
        d = F.decode(e)
        assert np.array_equal(d, p)                                 # decode . encode = id
        e2 = F.encode(d, fmt)                                       # encode . decode = id
        assert np.array_equal(e2.values, e.values) and np.array_equal(e2.codes, e.codes) \
            and np.array_equal(e2.idx, e.idx)
        assert np.count_nonzero(d) <= rows * cols * fmt.density
        # invariants: every kept 4-group has 2 strictly increasing codes
        c = e.codes.reshape(-1, 2)
        assert (c[:, 0] < c[:, 1]).all()


def test_pattern_errors():
    f = F.SparseFormat(1, 2, 4)
    with pytest.raises(F.PatternError):
        F.encode(bits([[1, 0, 0, 0], [1, 0, 0, 0]]), f)             # two sub-rows
    with pytest.raises(F.PatternError):
        F.encode(bits([[1, 1, 1, 0], [0, 0, 0, 0]]), f)             # 3 of 4
    with pytest.raises(F.ShapeError):
        F.encode(bits([[1, 0, 0]]), f)


def test_validate_detects_corruption():
    f = F.SparseFormat(1, 2, 4)
    e = F.encode(bits([[1, 0, 2, 0], [0, 0, 0, 0]]), f)
    e.codes[0] = [3, 1]
    assert any(v[0] == "metadata_not_increasing" for v in F.validate(e))
    with pytest.raises(F.CorruptFormat):
        F.decode(e)
    e = F.encode(bits([[1, 0, 2, 0], [0, 0, 0, 0]]), f)
    e.idx[0, 0] = 2
    assert any(v[0] == "index_out_of_range" for v in F.validate(e))


def test_fill_rule_lowest_unused():
    f = F.SparseFormat(2, 4, 4)
    w = np.zeros((4, 4))
    w[2] = [0, 5, 0, 6]
    e = F.encode(bits(w), f)
    assert e.idx[:, 0].tolist() == [0, 2]                           # R5: fill with row 0


# ------------------------------------------------------------- packing

def test_panel_golden_and_bijection():
    for (src, dst) in GOLD["pack_panel_map"]["pairs"]:
        m = np.zeros((16, 16), dtype=np.int64)
        m[src[0], src[1]] = 7
        p = F.pack_panel(m)
        assert p[dst[0], dst[1]] == 7 and p.sum() == 7
    rng = np.random.default_rng(4)
    for _ in range(200):
        m = rng.integers(0, 4, (16, 16))
        assert np.array_equal(F.unpack_panel(F.pack_panel(m)), m)
    # bijection: the map is a permutation of the 256 positions
    tgt = {(r % 8 * 2 + c // 8, c % 8 + r // 8 * 8) for r in range(16) for c in range(16)}
    assert len(tgt) == 256


def test_pack_codes_roundtrip_and_bit_order():
    c = np.array([[1, 2, 3, 0, 0, 1, 2, 3]], dtype=np.uint8)
    p = F.pack_codes(c)
    assert p.tolist() == [[1 | 2 << 2 | 3 << 4, 0 | 1 << 2 | 2 << 4 | 3 << 6]]
    rng = np.random.default_rng(5)
    c = rng.integers(0, 4, (9, 64)).astype(np.uint8)
    assert np.array_equal(F.unpack_codes(F.pack_codes(c)), c)


# ------------------------------------------------------------- sizes

def test_memreport_closed_form():
    g = GOLD["memreport_1408x2048_f32_1_2_16"]
    b = F.canonical_bytes(g["rows"], g["cols"], F.SparseFormat(*g["fmt"]), g["elem_bytes"])
    for k in ("dense", "values", "codes", "indices"):
        assert b[k] == g[k]
    ratio = (b["values"] + b["codes"] + b["indices"]) / b["dense"] * 100
    assert abs(ratio - g["ratio_percent"]) < 0.005


def test_bytes_per_element_bf16():
    g = GOLD["bytes_per_elem_bf16_1_2_32"]
    b = F.canonical_bytes(4096, 14336, F.SparseFormat(*g["fmt"]), 2)
    per = (b["values"] + b["codes"] + b["indices"]) / (4096 * 14336)
    assert per == g["bytes_per_logical_element"]


# ------------------------------------------------ interleaved gate/up (R20)

@pytest.mark.parametrize("fmt", list(F.TABLE4) + [F.SparseFormat(2, 2, 32)])
def test_interleave_commutes_with_prune_and_encode(fmt):
    """Pruning and encoding act on M-row groups and 128 is a multiple of every
    M, so encoding the interleaved dense weight must give exactly the
    interleaved encodings (a wrong block size, offset or row order breaks it)."""
    f, d = 256, 128
    wg = synth.weight_bf16(71, f, d)
    wu = synth.weight_bf16(72, f, d)
    direct = F.encode(F.prune(F.interleave_rows(wg, wu, F.gu_block(fmt)), fmt), fmt)
    built = F.interleave_gate_up(F.encode(F.prune(wg, fmt), fmt), F.encode(F.prune(wu, fmt), fmt))
    assert (direct.rows, direct.cols) == (built.rows, built.cols) == (2 * f, d)
    for name in ("values", "codes", "idx"):
        assert np.array_equal(getattr(direct, name), getattr(built, name)), name


def test_interleave_rows_layout_and_inverse():
    f, d = 96, 8
    wg = np.arange(f * d, dtype=np.uint16).reshape(f, d)
    wu = wg + np.uint16(10000)
    assert F.GU_BLOCK == 32 and F.gu_block(F.SparseFormat(1, 2, 32)) == 32 and F.gu_block(F.SparseFormat(2, 2, 32)) == 16
    assert F.gu_block(F.SparseFormat(4, 8, 32)) == 32
    gu = F.interleave_rows(wg, wu)
    # row 32 of the interleaved weight is up row 0; row 64 is gate row 32
    assert np.array_equal(gu[0], wg[0]) and np.array_equal(gu[31], wg[31])
    assert np.array_equal(gu[32], wu[0]) and np.array_equal(gu[63], wu[31])
    assert np.array_equal(gu[64], wg[32]) and np.array_equal(gu[191], wu[95])
    g2, u2 = F.deinterleave_rows(gu)
    assert np.array_equal(g2, wg) and np.array_equal(u2, wu)
    with pytest.raises(F.ShapeError):
        F.interleave_rows(wg[:40], wu[:40])
