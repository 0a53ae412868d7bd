"""Pins for oracle/devlayout.py, oracle/ssmm.py and oracle/moe.py (CPU only)."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import bf16, devlayout as D, fmt as F, moe, ssmm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bits(a):
    return synth.f32_to_bf16_bits(np.asarray(a, dtype=np.float32))


def make_enc(fmt, rows, cols, seed=11, integer=False):
    w = synth.weight_bf16(seed, rows, cols, integer=integer)
    return F.encode(F.prune(w, fmt), fmt)


# ----------------------------------------------------------- device layouts

@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 32), F.SparseFormat(1, 2, 16), F.SparseFormat(4, 8, 32)])
def test_a_image_is_sw128_permutation_of_values(fmt):
    enc = make_enc(fmt, 192 * fmt.m // fmt.n // 2 * 2, 256)
    img = D.a_image(enc)
    g = D.geometry(enc.rows, enc.cols, fmt)
    # independent formulation of the 128B swizzle: byte offset bits [4,7) ^= bits [7,10)
    rep = g["rep"]
    for t in range(g["m_tiles"]):
        for s in range(g["k_stages"]):
            blk = img[t, s]
            for r in (0, 5, 63, 127):
                cr = t * 128 + r
                for c in range(64):
                    lin = r * 128 + c * 2
                    phys = lin ^ (((lin >> 7) & 7) << 4)
                    got = blk[phys:phys + 2].view(np.uint16)[0]
                    vb, slot = s * 4 + c // 16, c % 16
                    if cr >= g["R"]:
                        assert got == 0
                        continue
                    j, h = vb // rep, vb % rep
                    if rep == 1 or (slot // 8) == h:
                        assert got == enc.values[cr, j * 16 + slot]
                    else:
                        assert got == 0


def test_e_image_matches_cutlass_atom_formula():
    """The TMEM-image lane order must equal the sm1xx sparse E atom
    (TensorEAtom_MMA_F16 Shape((8,2,8),(16,2,4)):Stride((128,16,2048),(1,1024,32)),
    in 8-logical-element bytes) -- an independent derivation."""
    fmt = F.SparseFormat(1, 2, 32)
    enc = make_enc(fmt, 256, 256)
    img = D.e_image(enc)                                   # [mt, ks, 2048]
    for t in range(img.shape[0]):
        for s in range(img.shape[1]):
            blk = img[t, s]
            for m in range(128):
                cr = t * 128 + m
                for k in range(0, 128, 4):                  # logical K within the stage
                    byte = (256 * (m // 16) + 128 * ((k // 16) % 2) + 16 * (m % 8) + 4 * (k // 32)
                            + 2 * ((m // 8) % 2) + (k % 16) // 8)
                    nib = (blk[byte] >> (4 * ((k % 8) // 4))) & 0xF
                    q = (s * 128 + k) // 4                  # 4-group index along the row
                    p0, p1 = enc.codes[cr, 2 * q], enc.codes[cr, 2 * q + 1]
                    assert nib == (p0 | (p1 << 2))


def test_planes_bits():
    fmt = F.SparseFormat(4, 8, 32)
    enc = make_enc(fmt, 512, 256)
    P = D.n_planes(fmt)
    assert P == 3
    pl = D.planes(enc)
    mt, ks = pl.shape[:2]
    words = np.ascontiguousarray(pl).view(np.uint32).reshape(mt, ks, 4, P, 4)
    for t in range(mt):
        for s in range(ks):
            for kb in range(4):
                for lane in range(128):
                    v = enc.idx[t * 128 + lane, s * 4 + kb]
                    got = sum(((int(words[t, s, kb, b, lane // 32]) >> (lane % 32)) & 1) << b for b in range(P))
                    assert got == v
    assert D.n_planes(F.SparseFormat(2, 2, 32)) == 0 and D.n_planes(F.SparseFormat(1, 2, 32)) == 1


# ---------------------------------------------------------------- SSMM

@pytest.mark.parametrize("fmt", F.TABLE4)
def test_ssmm_equals_brute_force_masked_matmul(fmt):
    rows, cols = 2 * fmt.m, 64
    w = F.prune(synth.weight_bf16(21, rows, cols), fmt)
    x = synth.activations_bf16(22, 12, cols)
    sel = np.array([0, 3, 4, 11])
    enc = F.encode(w, fmt)
    got = ssmm.ssmm(enc, x, sel)
    ref = ssmm.masked_dense_reference(w, x, sel)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_ssmm_identity_pattern_selects_x():
    fmt = F.SparseFormat(1, 2, 32)
    rows, cols = 4, 4 * 32
    w = np.zeros((rows, cols))
    for o in range(rows):
        w[o, 32 * o] = 1.0
    enc = F.encode(bits(w), fmt)
    x = synth.activations_bf16(3, 9, cols)
    sel = np.array([1, 2, 8])
    c = ssmm.ssmm(enc, x, sel)
    assert np.array_equal(c, bf16.to_f64(x)[sel][:, [0, 32, 64, 96]])
    assert ssmm.ssmm(enc, x, np.array([], dtype=np.int64)).shape == (0, rows)


def test_ssmm_integer_inputs_exact_and_linear():
    fmt = F.SparseFormat(1, 2, 32)
    enc = make_enc(fmt, 64, 128, integer=True)
    x = synth.activations_bf16(5, 16, 128, integer=True)
    sel = np.arange(16)
    c = ssmm.ssmm(enc, x, sel)
    assert np.array_equal(c, np.round(c))
    x2 = synth.activations_bf16(6, 16, 128, integer=True)
    xs = bits(bf16.to_f64(x) + bf16.to_f64(x2))
    assert np.array_equal(ssmm.ssmm(enc, xs, sel), c + ssmm.ssmm(enc, x2, sel))


def test_epilogues():
    fmt = F.SparseFormat(1, 2, 32)
    g, u = make_enc(fmt, 64, 128, 1), make_enc(fmt, 64, 128, 2)
    x = synth.activations_bf16(7, 10, 128)
    sel = np.array([2, 5, 9])
    cg, cu = ssmm.ssmm(g, x, sel), ssmm.ssmm(u, x, sel)
    a = ssmm.silu_mul_bf16(cg, cu)
    ref = cg / (1 + np.exp(-cg)) * cu
    assert np.all(np.abs(bf16.to_f64(a) - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-30)
    out = ssmm.scatter_add(np.zeros((10, 64)), cg, sel, [0.5, 2.0, -1.0])
    assert np.array_equal(out[5], 2.0 * cg[1]) and np.array_equal(out[0], np.zeros(64))


# ---------------------------------------------------------------- routing

def test_route_golden_and_invariants():
    for case in GOLD["route"]["cases"]:
        ids, w = moe.route(np.array([case["logits"]], dtype=np.float32), case["k"])
        assert ids[0].tolist() == case["ids"]
        assert np.allclose(w[0], case["w"])
    lg = synth.router_logits(2, 50, 8)
    ids, w = moe.route(lg, 2)
    assert np.allclose(w.sum(1), 1.0, atol=1e-12)
    ids2, w2 = moe.route(lg + np.float32(3.0), 2)                    # shift invariance (exact in fp32 here?)
    assert np.array_equal(ids, ids2)
    ids3, w3 = moe.route(lg, 2, moe.SOFTMAX_ALL)
    assert np.array_equal(ids, ids3) and (w3.sum(1) < 1).all()


def test_route_gate_weights_closed_form():
    """Hand-computed gate weights (P:151 weighted sum; readings R9, R10): with
    logits ln(c_e) the softmax of a subset is c_e / sum(c).  Pins the SOFTMAX_ALL
    weights (denominator over ALL E, values taken at the selected ids) and
    RENORM_TOPK (denominator over the selected k) -- a wrong index into the
    exponentials (e.g. the first k instead of the selected ones) fails."""
    lg = np.log(np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0]], dtype=np.float64)).astype(np.float32)
    ids, w = moe.route(lg, 2, moe.SOFTMAX_ALL)
    assert ids[0].tolist() == [2, 1]
    assert np.allclose(w[0], [3 / 6, 2 / 6], rtol=1e-6, atol=0)
    ids, w = moe.route(lg, 2, moe.RENORM_TOPK)
    assert ids[0].tolist() == [2, 1]
    assert np.allclose(w[0], [3 / 5, 2 / 5], rtol=1e-6, atol=0)
    # E = 5, k = 3, selected ids not a prefix: c = [4, 1, 5, 2, 3]
    c = np.array([4.0, 1.0, 5.0, 2.0, 3.0])
    lg = np.log(c)[None, :].astype(np.float32)
    ids, w = moe.route(lg, 3, moe.SOFTMAX_ALL)
    assert ids[0].tolist() == [2, 0, 4]
    assert np.allclose(w[0], [5 / 15, 4 / 15, 3 / 15], rtol=1e-6, atol=0)
    ids, w = moe.route(lg, 3, moe.RENORM_TOPK)
    assert np.allclose(w[0], [5 / 12, 4 / 12, 3 / 12], rtol=1e-6, atol=0)
    # a NaN logit ranks as -inf (R10b): selected after every finite logit, weight 0
    lg = np.array([[np.nan, np.log(2.0), 0.0, np.nan]], dtype=np.float32)
    ids, w = moe.route(lg, 3, moe.SOFTMAX_ALL)
    assert ids[0].tolist() == [1, 2, 0] and np.allclose(w[0], [2 / 3, 1 / 3, 0.0], rtol=1e-6, atol=0)
    ids, w = moe.route(lg, 2, moe.RENORM_TOPK)
    assert ids[0].tolist() == [1, 2] and np.allclose(w[0], [2 / 3, 1 / 3], rtol=1e-6, atol=0)
    # ties -> lower id (R10), weights equal
    ids, w = moe.route(np.zeros((1, 4), dtype=np.float32), 2, moe.SOFTMAX_ALL)
    assert ids[0].tolist() == [0, 1] and np.allclose(w[0], [0.25, 0.25], rtol=1e-12)


def _bf16_rne(v: float) -> float:
    """Round-to-nearest-even to 8 significant bits, written out (independent of
    oracle/bf16.py): v = q * 2^(e-8) with q scaled to [128, 256); Python's
    round() is round-half-even and q is exact in fp64."""
    import math
    if v == 0.0:
        return 0.0
    _, e = math.frexp(v)               # v = m * 2^e, 0.5 <= |m| < 1
    step = math.ldexp(1.0, e - 8)
    return round(v / step) * step


def test_layer_error_scale_brute_force():
    """The per-element error scale S of the layer (north star: |err| <= 1e-2 *
    sum |g * w * a|), pinned from above and below by an element loop over the
    pruned dense weights: S[t,o] = sum_(e,g in route(t)) |g| sum_j |Wd_e[o,j]|
    |a_e[t,j]|, with a_e[t] = bf16(silu(Wg_e x_t) * (Wu_e x_t)) -- and the
    output itself, same loop, for good measure."""
    import math
    fmt = F.SparseFormat(1, 2, 32)
    E, d, f, T, k = 3, 64, 64, 4, 2
    dense = []
    for e in range(E):
        trip = []
        for i in range(3):
            r, c = (f, d) if i < 2 else (d, f)
            trip.append(bf16.to_f64(F.prune(synth.weight_bf16(700 + 3 * e + i, r, c), fmt)))
        dense.append(trip)
    ex = [tuple(F.encode(F.prune(synth.weight_bf16(700 + 3 * e + i, *((f, d) if i < 2 else (d, f))), fmt), fmt)
                for i in range(3)) for e in range(E)]
    xb = synth.activations_bf16(5, T, d)
    x = bf16.to_f64(xb)
    lg = synth.router_logits(6, T, E)
    for mode in (moe.RENORM_TOPK, moe.SOFTMAX_ALL):
        out, S = moe.moe_layer(ex, xb, lg, k, mode)
        out_bf = np.zeros((T, d))
        S_bf = np.zeros((T, d))
        for t in range(T):
            l = [float(v) for v in lg[t]]
            order = sorted(range(E), key=lambda e: (-l[e], e))[:k]
            den = sum(math.exp(l[e] - max(l)) for e in (order if mode == moe.RENORM_TOPK else range(E)))
            for e in order:
                g = math.exp(l[e] - max(l)) / den
                wg, wu, wd = dense[e]
                a = []
                for j in range(f):
                    h = sum(wg[j, c] * x[t, c] for c in range(d))
                    u = sum(wu[j, c] * x[t, c] for c in range(d))
                    a.append(_bf16_rne(h / (1.0 + math.exp(-h)) * u))
                for o in range(d):
                    out_bf[t, o] += g * sum(wd[o, j] * a[j] for j in range(f))
                    S_bf[t, o] += abs(g) * sum(abs(wd[o, j] * a[j]) for j in range(f))
        assert np.allclose(S, S_bf, rtol=1e-9, atol=0), np.abs(S / S_bf - 1).max()
        assert np.allclose(out, out_bf, rtol=1e-9, atol=1e-12)


def test_compaction_partition():
    lg = synth.router_logits(2, 64, 8)
    ids, w = moe.route(lg, 2)
    counts, offsets, sel, gw = moe.compact(ids, w, 8)
    assert counts.sum() == 64 * 2
    for e in range(8):
        s = sel[offsets[e]:offsets[e + 1]]
        assert (np.diff(s) > 0).all()                                # strictly ascending
        for t in s:
            assert e in ids[t]
    pairs = {(int(t), e) for e in range(8) for t in sel[offsets[e]:offsets[e + 1]]}
    assert pairs == {(t, int(e)) for t in range(64) for e in ids[t]}


# ---------------------------------------------------------------- layer

def _experts(fmt, E, d, f, seed0=1000, integer=False):
    ex = []
    for e in range(E):
        ex.append(tuple(make_enc(fmt, *(f, d) if i < 2 else (d, f), seed=seed0 + 3 * e + i, integer=integer)
                        for i in range(3)))
    return ex


def test_layer_equals_textbook_permute_gemm_unpermute():
    fmt = F.SparseFormat(1, 2, 32)
    E, d, f, T, k = 4, 64, 96, 20, 2
    ex = _experts(fmt, E, d, f)
    x = synth.activations_bf16(1, T, d)
    lg = synth.router_logits(2, T, E)
    out, S = moe.moe_layer(ex, x, lg, k)
    dense = [tuple(F.dense_f64(w) for w in trip) for trip in ex]
    ref = moe.moe_layer_textbook(dense, x, lg, k)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    perm = np.random.default_rng(0).permutation(T)
    out_p, _ = moe.moe_layer(ex, x[perm], lg[perm], k)
    assert np.allclose(out_p, out[perm], rtol=1e-12, atol=1e-12)
    z, _ = moe.moe_layer(ex, np.zeros_like(x), lg, k)
    assert not z.any()
    assert (S >= np.abs(out) - 1e-12).all()


def test_layer_all_tokens_one_expert_and_shared():
    fmt = F.SparseFormat(1, 2, 32)
    E, d, f, T = 2, 64, 64, 6
    ex = _experts(fmt, E, d, f)
    x = synth.activations_bf16(1, T, d)
    lg = np.zeros((T, E), dtype=np.float32)
    lg[:, 0] = 5.0
    out, _ = moe.moe_layer(ex, x, lg, 1)
    y, _, _ = moe.expert_ffn(*ex[0], x, np.arange(T))
    assert np.allclose(out, y, rtol=1e-12, atol=1e-12)
    sh = _experts(fmt, 2, d, f, seed0=5000)
    out2, _ = moe.moe_layer(ex, x, lg, 1, shared=sh)
    y0, _, _ = moe.expert_ffn(*sh[0], x, np.arange(T))
    y1, _, _ = moe.expert_ffn(*sh[1], x, np.arange(T))
    assert np.allclose(out2, y + y0 + y1, rtol=1e-12, atol=1e-12)


def test_layer_sigmoid_gated_shared_expert():
    """Reading R15b (Qwen2-MoE's shared expert, scaled per token by the sigmoid of
    a shared-gate logit): closed-form gates sigmoid(0) = 1/2, sigmoid(ln 3) = 3/4,
    sigmoid(-ln 3) = 1/4, and the decomposition the bench relies on -- one shared
    FFN of width 2f equals two width-f shared experts under the same gate, computed
    here as the wide FFN from the decoded dense weights."""
    fmt = F.SparseFormat(1, 2, 32)
    E, d, f, T = 2, 64, 64, 3
    ex = _experts(fmt, E, d, f)
    x = synth.activations_bf16(1, T, d)
    lg = np.zeros((T, E), dtype=np.float32)
    lg[:, 0] = 5.0
    y, _, _ = moe.expert_ffn(*ex[0], x, np.arange(T))
    sh = _experts(fmt, 2, d, f, seed0=5000)
    z = np.array([[0.0, 0.0], [np.log(3.0), np.log(3.0)], [-np.log(3.0), -np.log(3.0)]], dtype=np.float32)
    out, S = moe.moe_layer(ex, x, lg, 1, shared=sh, shared_logits=z)
    xf = bf16.to_f64(x)
    g = xf @ np.vstack([F.dense_f64(sh[0][0]), F.dense_f64(sh[1][0])]).T       # [T x 2f]
    u = xf @ np.vstack([F.dense_f64(sh[0][1]), F.dense_f64(sh[1][1])]).T
    a = bf16.to_f64(bf16.from_f64(g / (1.0 + np.exp(-g)) * u))
    wide = a @ np.hstack([F.dense_f64(sh[0][2]), F.dense_f64(sh[1][2])]).T      # [T x d]
    c = np.array([0.5, 0.75, 0.25])
    assert np.allclose(out[0], y[0] + 0.5 * wide[0], rtol=1e-12, atol=1e-12)      # z = 0 exactly
    assert np.allclose(out, y + c[:, None] * wide, rtol=0, atol=1e-7)           # ln 3 rounded to fp32
    out1, S1 = moe.moe_layer(ex, x, lg, 1, shared=sh)
    assert np.allclose(out1, y + wide, rtol=1e-12, atol=1e-12)                 # ungated: weight 1 (R15)
    assert (S <= S1 + 1e-12).all() and (S >= np.abs(out) - 1e-12).all()


def test_ep_plan_covers_routing_once():
    E, P, T, k = 8, 4, 16, 2
    ids_r, w_r = [], []
    for s in range(P):
        ids, w = moe.route(synth.router_logits(100 + s, T, E), k)
        ids_r.append(ids)
        w_r.append(w)
    recv = moe.ep_dispatch_plan(ids_r, w_r, E, P)
    seen = set()
    for d in range(P):
        keys = [(s, t) for s, t, _ in recv[d]]
        assert keys == sorted(keys) and len(set(keys)) == len(keys)
        for s, t, tags in recv[d]:
            for le, _ in tags:
                seen.add((s, t, d * (E // P) + le))
    assert seen == {(s, t, int(e)) for s in range(P) for t in range(T) for e in ids_r[s][t]}


def test_silu_mul_interleaved_equals_two_weight_epilogue():
    """One SSMM on the interleaved gate/up weight + the interleaved epilogue
    equals the two-weight SILU_MUL path bit for bit (same fp64 arithmetic)."""
    fmt = F.SparseFormat(1, 2, 32)
    eg, eu = make_enc(fmt, 256, 128, seed=81), make_enc(fmt, 256, 128, seed=82)
    x = synth.activations_bf16(83, 40, 128)
    sel = np.array([0, 3, 4, 9, 17, 21, 39], dtype=np.int32)
    gu = F.interleave_gate_up(eg, eu)
    got = ssmm.silu_mul_interleaved_bf16(ssmm.ssmm(gu, x, sel))
    ref = ssmm.silu_mul_bf16(ssmm.ssmm(eg, x, sel), ssmm.ssmm(eu, x, sel))
    assert got.shape == (len(sel), 256)
    assert np.array_equal(got, ref)
