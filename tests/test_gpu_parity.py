"""GPU parity tests: CUDA path (through the C ABI) vs the fp64 CPU oracle.

Bars (BASELINE.json north star): compressor / metadata / routing indices
bit-exact; SSMM and layer outputs within relative Frobenius 1e-3 and
per-element |err| <= 1e-2 * sum|w*x|; integer-valued inputs bit-exact.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import bf16, devlayout as D, fmt as F, moe, ssmm as OS

pytestmark = pytest.mark.gpu

REL_FRO = 1e-3
ELEM = 1e-2


@pytest.fixture(scope="module")
def smy():
    import paper_2503_10725_b200 as P
    P.load()
    return P


def dev16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda()


def host16(t):
    return t.cpu().numpy().view(np.uint16)


def gpu_format(fmt):
    from paper_2503_10725_b200 import Format
    return Format(fmt.n, fmt.m, fmt.v)


def check_tol(got, ref, scale, what):
    err = np.abs(got - ref)
    rf = OS.rel_fro(got - ref, ref)
    bad = err > ELEM * scale + 1e-30
    assert rf <= REL_FRO, f"{what}: rel Frobenius {rf:.3e} > {REL_FRO}"
    assert not bad.any(), f"{what}: {bad.sum()} elements beyond 1e-2*sum|wx|, first at {np.argwhere(bad)[:3]}"


def bf16_ulp(v):
    """one bf16 ulp at |v| (8 significant bits); 0 at v = 0"""
    a = np.abs(v)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, np.exp2(e - 7), 0.0)


def check_silu_mul(got, cg, cu, Sg, Su, what):
    """The gate/up intermediate at the north-star bar against the oracle's bf16
    output bf16(silu(C_g) * C_u) (P:337 fused activation, R12 bf16 intermediate):
    rel Frobenius <= 1e-3 and EVERY element within one bf16 ulp (the two
    roundings of the stored value) plus the 1e-2 * sum|w*x| bound on C_g / C_u
    propagated through silu(g) * u: |silu'(g) u| * 1e-2 S_g + |silu(g)| * 1e-2 S_u."""
    ref = bf16.to_f64(OS.silu_mul_bf16(cg, cu))
    sig = 1.0 / (1.0 + np.exp(-cg))
    dsilu = sig * (1.0 + cg * (1.0 - sig))
    bound = (np.maximum(bf16_ulp(ref), bf16_ulp(got)) + ELEM * (np.abs(dsilu * cu) * Sg + np.abs(cg * sig) * Su)
             + 1e-30)
    rf = OS.rel_fro(got - ref, ref)
    assert rf <= REL_FRO, f"{what}: rel Frobenius {rf:.3e} > {REL_FRO}"
    bad = np.abs(got - ref) > bound
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} elements beyond the bound, first at {np.argwhere(bad)[:3]}"


PARITY_FORMATS = [F.SparseFormat(1, 2, 32), F.SparseFormat(1, 2, 16), F.SparseFormat(4, 8, 32),
                  F.SparseFormat(8, 16, 32), F.SparseFormat(2, 2, 32), F.SparseFormat(1, 1, 32)]


# ------------------------------------------------------------------ synth twin

def test_synth_twin_bit_exact(smy):
    n, idx0 = 5000, 12345
    idx = np.arange(idx0, idx0 + n, dtype=np.uint64)
    for dist, scale in ((synth.DIST_UNIFORM, synth.uniform_scale(0.05)), (synth.DIST_NORMAL, synth.normal_scale(1.0)),
                        (synth.DIST_INT, 0.0)):
        ref = synth.fill_f32(77, idx, dist, scale)
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        smy.synth_fill(t, 77, dist, float(scale), idx0=idx0)
        assert np.array_equal(t.cpu().numpy().view(np.uint32), ref.view(np.uint32)), dist
        tb = torch.empty(n, dtype=torch.int16, device="cuda")
        smy.synth_fill(tb, 77, dist, float(scale), idx0=idx0)
        assert np.array_equal(host16(tb), synth.f32_to_bf16_bits(ref)), dist


# ------------------------------------------------------------------ compressor

@pytest.mark.parametrize("fmt", PARITY_FORMATS, ids=str)
def test_compress_bit_exact(smy, fmt):
    rows, cols = 256, 256
    w = synth.weight_bf16(31, rows, cols)
    enc = F.encode(F.prune(w, fmt), fmt)
    sw, status = smy.compress(dev16(w), gpu_format(fmt), prune=True)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert np.array_equal(host16(sw.values).reshape(enc.values.shape), enc.values)
    assert np.array_equal(sw.codes.cpu().numpy().reshape(-1, cols // 8), F.pack_codes(enc.codes))
    assert np.array_equal(sw.indices.cpu().numpy().reshape(enc.idx.shape), enc.idx)
    assert np.array_equal(sw.image.cpu().numpy(), D.weight_image(enc))
    # ASSUME_PRUNED on the oracle-pruned weight encodes identically
    sw2, st2 = smy.compress(dev16(F.prune(w, fmt)), gpu_format(fmt), prune=False)
    torch.cuda.synchronize()
    assert int(st2.item()) == 0
    assert torch.equal(sw2.image, sw.image) and torch.equal(sw2.values, sw.values)


def test_compress_pattern_error(smy):
    fmt = F.SparseFormat(1, 2, 32)
    w = synth.weight_bf16(3, 128, 128)                 # dense: violates the pattern
    _, status = smy.compress(dev16(w), gpu_format(fmt), prune=False)
    torch.cuda.synchronize()
    assert int(status.item()) == 4                     # SMY_E_PATTERN


def test_compress_rejects_bad_shapes(smy):
    from paper_2503_10725_b200 import SamoyedsError
    with pytest.raises(SamoyedsError):
        smy.compress(torch.zeros(128, 96, dtype=torch.int16, device="cuda"), smy.Format(1, 2, 32))


# ------------------------------------------------------------------ SSMM

def _ssmm_case(smy, fmt, rows, cols, x_rows, sel, integer, seed=41):
    w = synth.weight_bf16(seed, rows, cols, integer=integer)
    enc = F.encode(F.prune(w, fmt), fmt)
    x = synth.activations_bf16(seed + 1, x_rows, cols, integer=integer)
    sw, _ = smy.compress(dev16(w), gpu_format(fmt))
    return enc, x, sw


def test_ssmm_probe_identity_activations(smy):
    """E-metadata / A-layout probe: with x = identity, C = W^T exactly, so any
    mis-read of values, metadata or the sub-row remap shows up positionally."""
    fmt = F.SparseFormat(1, 2, 32)
    rows, cols = 256, 128
    w = synth.weight_bf16(5, rows, cols, integer=True)
    pruned = F.prune(w, fmt)
    enc = F.encode(pruned, fmt)
    x = synth.f32_to_bf16_bits(np.eye(cols, dtype=np.float32))
    sel = np.arange(cols, dtype=np.int32)
    sw, _ = smy.compress(dev16(w), gpu_format(fmt))
    c = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy()     # [cols x rows] = W^T
    ref = bf16.to_f64(pruned).T
    if not np.array_equal(c, ref):
        bad = np.argwhere(c != ref)
        lines = []
        for k, o in bad[:12]:
            hits = np.argwhere(c[:, o] == ref[k, o])[:4].ravel().tolist() if ref[k, o] != 0 else []
            lines.append(f"(k={k}, o={o}) got {c[k, o]} want {ref[k, o]}; value found at k={hits}")
        pytest.fail(f"{len(bad)} wrong of {c.size}:\n" + "\n".join(lines))


@pytest.mark.parametrize("fmt", PARITY_FORMATS, ids=str)
def test_ssmm_integer_bit_exact_cfg1(smy, fmt):
    """BASELINE config 1: W 128x256, 64 tokens with 16 routed; integer inputs -> exact."""
    sel = synth.selection(4, 64, 16)
    enc, x, sw = _ssmm_case(smy, fmt, 128, 256, 64, sel, integer=True)
    got = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy()
    ref = OS.ssmm(enc, x, sel)
    assert np.array_equal(got, ref), f"max |err| {np.abs(got - ref).max()}"


@pytest.mark.parametrize("fmt", PARITY_FORMATS, ids=str)
@pytest.mark.parametrize("shape", [(128, 256, 64, 16), (384, 512, 300, 200), (1024, 1408, 900, 777),
                                   (256, 512, 400, 110)])
def test_ssmm_random_tolerance(smy, fmt, shape):
    rows, cols, x_rows, n_sel = shape
    if cols % 128:
        pytest.skip("cols must be a multiple of 128")
    sel = synth.selection(9, x_rows, n_sel)
    enc, x, sw = _ssmm_case(smy, fmt, rows, cols, x_rows, sel, integer=False)
    got = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy().astype(np.float64)
    check_tol(got, OS.ssmm(enc, x, sel), OS.ssmm_abs(enc, x, sel), f"ssmm {fmt} {shape}")


def test_ssmm_ragged_and_empty(smy):
    fmt = F.SparseFormat(1, 2, 32)
    for n_sel in (0, 1, 15, 17, 113, 225, 449):
        sel = synth.selection(n_sel + 1, 512, n_sel)
        enc, x, sw = _ssmm_case(smy, fmt, 256, 256, 512, sel, integer=True)
        got = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy()
        assert got.shape == (n_sel, 256)
        assert np.array_equal(got, OS.ssmm(enc, x, sel)), n_sel


def test_ssmm_bf16_out(smy):
    fmt = F.SparseFormat(1, 2, 32)
    sel = synth.selection(2, 128, 40)
    enc, x, sw = _ssmm_case(smy, fmt, 256, 256, 128, sel, integer=True)
    got = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda(), out_dtype=torch.bfloat16)
    assert np.array_equal(host16(got.view(torch.int16)), bf16.from_f64(OS.ssmm(enc, x, sel)))


@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 32), F.SparseFormat(4, 8, 32), F.SparseFormat(1, 2, 16),
                                 F.SparseFormat(2, 2, 32)], ids=str)
def test_ssmm_scatter_add_exact(smy, fmt):
    """Fused weighted accumulation: power-of-two scales, integer inputs -> exact."""
    sel = synth.selection(6, 200, 77)
    enc, x, sw = _ssmm_case(smy, fmt, 256, 384, 200, sel, integer=True)
    scale = np.array([2.0 ** (i % 5 - 2) for i in range(len(sel))], dtype=np.float32)
    base = np.round(np.random.default_rng(0).standard_normal((200, 256)) * 4).astype(np.float32)
    out = torch.from_numpy(base.copy()).cuda()
    smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda(), epi="scatter_add", scale=torch.from_numpy(scale).cuda(),
             out=out)
    ref = OS.scatter_add(base.astype(np.float64), OS.ssmm(enc, x, sel), sel, scale)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 32), F.SparseFormat(4, 8, 32), F.SparseFormat(1, 2, 16),
                                 F.SparseFormat(1, 1, 32)], ids=str)
def test_ssmm_silu_mul(smy, fmt):
    """Fused gate/up + SiLU*up -> bf16 compact intermediate (R11, R12)."""
    from paper_2503_10725_b200 import Format
    sel = synth.selection(8, 300, 130)
    x = synth.activations_bf16(12, 300, 512)
    wg, wu = synth.weight_bf16(50, 384, 512), synth.weight_bf16(51, 384, 512)
    eg, eu = F.encode(F.prune(wg, fmt), fmt), F.encode(F.prune(wu, fmt), fmt)
    sg, _ = smy.compress(dev16(wg), gpu_format(fmt))
    su, _ = smy.compress(dev16(wu), gpu_format(fmt))
    got = smy.ssmm(sg, dev16(x), torch.from_numpy(sel).cuda(), epi="silu_mul", w2=su)
    got = bf16.to_f64(host16(got.view(torch.int16)))
    cg, cu = OS.ssmm(eg, x, sel), OS.ssmm(eu, x, sel)
    check_silu_mul(got, cg, cu, OS.ssmm_abs(eg, x, sel), OS.ssmm_abs(eu, x, sel), f"silu_mul {fmt}")


@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 32), F.SparseFormat(1, 2, 16), F.SparseFormat(4, 8, 32),
                                 F.SparseFormat(2, 2, 32)], ids=str)
def test_interleave_gate_up_bit_exact(smy, fmt):
    """samoyeds_interleave_gate_up (reading R20) == the oracle's interleaved
    encoding + device image, and == compressing the interleaved dense weight."""
    f, d = 384, 256
    wg, wu = synth.weight_bf16(61, f, d), synth.weight_bf16(62, f, d)
    eg, eu = F.encode(F.prune(wg, fmt), fmt), F.encode(F.prune(wu, fmt), fmt)
    ref = F.interleave_gate_up(eg, eu)
    sg, _ = smy.compress(dev16(wg), gpu_format(fmt))
    su, _ = smy.compress(dev16(wu), gpu_format(fmt))
    gu = smy.interleave_gate_up(sg, su)
    torch.cuda.synchronize()
    assert (gu.rows, gu.cols) == (2 * f, d)
    assert np.array_equal(host16(gu.values).reshape(ref.values.shape), ref.values)
    assert np.array_equal(gu.codes.cpu().numpy().reshape(-1, d // 8), F.pack_codes(ref.codes))
    assert np.array_equal(gu.indices.cpu().numpy().reshape(ref.idx.shape), ref.idx)
    assert np.array_equal(gu.image.cpu().numpy(), D.weight_image(ref))
    direct, _ = smy.compress(dev16(F.interleave_rows(wg, wu, F.gu_block(fmt))), gpu_format(fmt))
    assert torch.equal(direct.image, gu.image)


@pytest.mark.parametrize("shape", [(256, 256, 64, 16), (384, 512, 300, 130), (640, 512, 1000, 900)])
def test_ssmm_silu_mul_interleaved(smy, shape):
    """One SSMM over the interleaved gate/up weight with the fused SiLU*up
    epilogue (TMEM lanes l / l+64 paired through shared memory) vs the oracle;
    it must also equal the two-weight fused path bit for bit (same K order)."""
    f, d, x_rows, n_sel = shape
    fmt = F.SparseFormat(1, 2, 32)
    sel = synth.selection(8, x_rows, n_sel)
    x = synth.activations_bf16(12, x_rows, d)
    wg, wu = synth.weight_bf16(50, f, d), synth.weight_bf16(51, f, d)
    eg, eu = F.encode(F.prune(wg, fmt), fmt), F.encode(F.prune(wu, fmt), fmt)
    sg, _ = smy.compress(dev16(wg), gpu_format(fmt))
    su, _ = smy.compress(dev16(wu), gpu_format(fmt))
    gu = smy.interleave_gate_up(sg, su)
    st = torch.from_numpy(sel).cuda()
    got_t = smy.ssmm(gu, dev16(x), st, epi="silu_mul_interleaved")
    assert tuple(got_t.shape) == (n_sel, f)
    two = smy.ssmm(sg, dev16(x), st, epi="silu_mul", w2=su)
    assert torch.equal(got_t.view(torch.int16), two.view(torch.int16))
    got = bf16.to_f64(host16(got_t.view(torch.int16)))
    ref_bits = OS.silu_mul_interleaved_bf16(OS.ssmm(F.interleave_gate_up(eg, eu), x, sel))
    cg, cu = OS.ssmm(eg, x, sel), OS.ssmm(eu, x, sel)
    assert np.array_equal(ref_bits, OS.silu_mul_bf16(cg, cu))
    check_silu_mul(got, cg, cu, OS.ssmm_abs(eg, x, sel), OS.ssmm_abs(eu, x, sel), f"silu_mul_interleaved {shape}")


@pytest.mark.parametrize("fmt", [F.SparseFormat(4, 8, 32), F.SparseFormat(8, 16, 32), F.SparseFormat(2, 4, 32)],
                         ids=str)
@pytest.mark.parametrize("shape", [(256, 256, 64, 16), (384, 512, 300, 130), (640, 512, 1000, 900)])
def test_ssmm_silu_mul_interleaved_expanded(smy, fmt, shape):
    """(N, 2N, 32) formats, N > 1: the interleaved gate/up SSMM runs the in-smem row
    expansion of the compressed image, held to the north-star bar
    against the oracle's bf16 SiLU*up.  (Not bit-equal to the lane-masked M-slot
    kernel: that one sums a group's N lanes in the epilogue, a different fp32
    association; both are checked against the oracle.)"""
    f, d, x_rows, n_sel = shape
    sel = synth.selection(8, x_rows, n_sel)
    x = synth.activations_bf16(12, x_rows, d)
    wg, wu = synth.weight_bf16(50, f, d), synth.weight_bf16(51, f, d)
    eg, eu = F.encode(F.prune(wg, fmt), fmt), F.encode(F.prune(wu, fmt), fmt)
    sg, _ = smy.compress(dev16(wg), gpu_format(fmt))
    su, _ = smy.compress(dev16(wu), gpu_format(fmt))
    gu = smy.interleave_gate_up(sg, su)
    st = torch.from_numpy(sel).cuda()
    got_t = smy.ssmm(gu, dev16(x), st, epi="silu_mul_interleaved")
    assert tuple(got_t.shape) == (n_sel, f)
    got = bf16.to_f64(host16(got_t.view(torch.int16)))
    cg, cu = OS.ssmm(eg, x, sel), OS.ssmm(eu, x, sel)
    assert np.array_equal(OS.silu_mul_interleaved_bf16(OS.ssmm(F.interleave_gate_up(eg, eu), x, sel)),
                          OS.silu_mul_bf16(cg, cu))
    check_silu_mul(got, cg, cu, OS.ssmm_abs(eg, x, sel), OS.ssmm_abs(eu, x, sel), f"expanded silu_mul {fmt} {shape}")


@pytest.mark.parametrize("fmt", [F.SparseFormat(4, 8, 32), F.SparseFormat(8, 16, 32), F.SparseFormat(2, 4, 32)],
                         ids=str)
@pytest.mark.parametrize("epi", ["compact", "scatter_add", "compact_bf16", "compact_longk"])
def test_ssmm_expanded_integer_exact(smy, fmt, epi):
    """The row-expansion kernel on integer inputs (exact): compact fp32 / bf16 and the
    weighted scatter-add, over several m-tiles with a partial last one (rows 640 ->
    320 compressed rows), ragged token tiles and K of 5 stages; compact_longk: few tiles
    and K = 2560 (20 stages), which samoyeds_ssmm runs as a split-K / stream-K
    scatter-add into zeroed rows."""
    rows, cols, x_rows, n_sel = 640, 640, 500, 333
    if epi == "compact_longk":
        rows, cols, x_rows, n_sel, epi = 256, 2560, 200, 40, "compact"
    sel = synth.selection(21, x_rows, n_sel)
    enc, x, sw = _ssmm_case(smy, fmt, rows, cols, x_rows, sel, integer=True)
    st = torch.from_numpy(sel).cuda()
    ref = OS.ssmm(enc, x, sel)
    if epi == "scatter_add":
        scale = np.array([2.0 ** (i % 5 - 2) for i in range(n_sel)], dtype=np.float32)
        base = np.round(np.random.default_rng(1).standard_normal((x_rows, rows)) * 4).astype(np.float32)
        out = torch.from_numpy(base.copy()).cuda()
        smy.ssmm(sw, dev16(x), st, epi="scatter_add", scale=torch.from_numpy(scale).cuda(), out=out)
        assert np.array_equal(out.cpu().numpy(), OS.scatter_add(base.astype(np.float64), ref, sel, scale))
    elif epi == "compact_bf16":
        got = smy.ssmm(sw, dev16(x), st, out_dtype=torch.bfloat16)
        assert np.array_equal(host16(got.view(torch.int16)), bf16.from_f64(ref))
    else:
        assert np.array_equal(smy.ssmm(sw, dev16(x), st).cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", PARITY_FORMATS, ids=str)
def test_decompress_and_transcode(smy, fmt):
    """samoyeds_decompress returns the oracle's pruned dense weight bit for bit;
    the plain-2:4 transcode (the fast path for N>1 / V=16 formats) gives the
    same SSMM as the original format on integer inputs (exact)."""
    rows, cols = 256, 256
    w = synth.weight_bf16(33, rows, cols, integer=True)
    sw, _ = smy.compress(dev16(w), gpu_format(fmt))
    dense = smy.decompress(sw)
    assert np.array_equal(host16(dense), F.prune(w, fmt))
    again, st = smy.compress(dense, gpu_format(fmt), prune=False)
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and torch.equal(again.image, sw.image)
    t24 = smy.transcode_24(sw)
    x = synth.activations_bf16(34, 200, cols, integer=True)
    sel = synth.selection(3, 200, 150)
    a = smy.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy()
    b = smy.ssmm(t24, dev16(x), torch.from_numpy(sel).cuda()).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(b, OS.ssmm(F.encode(F.prune(w, fmt), fmt), x, sel))


def test_ssmm_full_size_sampled(smy):
    """Mixtral gate_proj at full size (14336 x 4096), 1024 of 4096 tokens, in the
    launch configuration the layer uses; the oracle recomputes sampled output
    rows from regenerated weight rows (the generator is counter-based)."""
    fmt = F.SparseFormat(1, 2, 32)
    rows, cols, T, n_sel = 14336, 4096, 4096, 1024
    seed = synth.weight_seed(0, 0)
    wt = torch.empty(rows, cols, dtype=torch.int16, device="cuda")
    smy.synth_fill(wt, seed, synth.DIST_UNIFORM, float(synth.uniform_scale(np.sqrt(3.0 / cols))))
    xt = torch.empty(T, cols, dtype=torch.int16, device="cuda")
    smy.synth_fill(xt, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    sel = synth.selection(17, T, n_sel)
    sw, _ = smy.compress(wt, smy.Format(1, 2, 32))
    got = smy.ssmm(sw, xt, torch.from_numpy(sel).cuda()).cpu().numpy()
    del wt
    rng = np.random.default_rng(0)
    groups = rng.choice(rows // 2, 24, replace=False)
    x = synth.activations_bf16(synth.SEED_X, T, cols, row_idx=sel)          # only the routed rows
    for g in groups:
        wrows = synth.weight_bf16(seed, rows, cols, row_idx=[2 * g, 2 * g + 1])
        enc = F.encode(F.prune(wrows, fmt), fmt)
        ref = OS.ssmm(enc, x, np.arange(n_sel))
        S = OS.ssmm_abs(enc, x, np.arange(n_sel))
        check_tol(got[:, 2 * g:2 * g + 2].astype(np.float64), ref, S, f"row group {g}")


# ------------------------------------------------------------------ routing

@pytest.mark.parametrize("T,E,k,gating", [(1, 8, 2, "renorm_topk"), (1000, 64, 6, "renorm_topk"),
                                          (777, 64, 8, "softmax_all"), (4096, 8, 2, "renorm_topk"),
                                          (300, 60, 4, "renorm_topk"),
                                          # T <= 256: the single-launch path; E up to 256
                                          (16, 64, 6, "softmax_all"), (256, 160, 8, "renorm_topk"),
                                          (257, 256, 8, "softmax_all")])
def test_route_bit_exact(smy, T, E, k, gating):
    lg = synth.router_logits(synth.SEED_LOGITS, T, E, skew=1.0 if E == 64 else 0.0)
    ids, w, counts, offsets, sel, gw = smy.route(torch.from_numpy(lg).cuda(), k, gating)
    rid, rw = moe.route(lg, k, moe.SOFTMAX_ALL if gating == "softmax_all" else moe.RENORM_TOPK)
    rc, ro, rs, rg = moe.compact(rid, rw, E)
    assert np.array_equal(ids.cpu().numpy(), rid)
    assert np.array_equal(counts.cpu().numpy(), rc)
    assert np.array_equal(offsets.cpu().numpy(), ro)
    assert np.array_equal(sel.cpu().numpy(), rs)
    assert np.allclose(w.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)
    assert np.allclose(gw.cpu().numpy(), rg, rtol=2e-6, atol=1e-7)


def test_route_ties(smy):
    lg = np.zeros((64, 8), dtype=np.float32)
    lg[:, 3] = 1.0
    ids, *_ = smy.route(torch.from_numpy(lg).cuda(), 3)
    assert np.array_equal(ids.cpu().numpy(), moe.route(lg, 3)[0])      # ties -> lower ids


# ------------------------------------------------------------------ MoE layer

def _layer_case(smy, fmt, E, d, f, T, k, gating="renorm_topk", shared=0, skew=0.0, seed_off=0, gate_up="auto",
                transcode="auto", variant=None, shared_gate="none"):
    cfg = smy.MoEConfig(E, k, d, f, shared, gating, gpu_format(fmt), gate_up, transcode, shared_gate=shared_gate)
    encs, sws = [], []
    for e in range(E + shared):
        te, ts = [], []
        for i in range(3):
            r, c = (f, d) if i < 2 else (d, f)
            w = synth.weight_bf16(synth.weight_seed(e + seed_off, i), r, c)
            te.append(F.encode(F.prune(w, fmt), fmt))
            ts.append(smy.compress(dev16(w), gpu_format(fmt))[0])
        encs.append(tuple(te))
        sws.append(tuple(ts))
    x = synth.activations_bf16(synth.SEED_X, T, d)
    sig = shared_gate == "sigmoid"
    lg = synth.router_logits(synth.SEED_LOGITS, T, E + (shared if sig else 0), skew=skew)
    layer = smy.MoELayer(cfg, sws[:E], sws[E:], max_tokens=max(T, 1))
    if variant is None:
        got = layer(dev16(x), torch.from_numpy(lg).cuda()).cpu().numpy().astype(np.float64)
    else:
        with layer.variant(variant, T):
            got = layer(dev16(x), torch.from_numpy(lg).cuda()).cpu().numpy().astype(np.float64)
    mode = moe.SOFTMAX_ALL if gating == "softmax_all" else moe.RENORM_TOPK
    ref, S = moe.moe_layer(encs[:E], x, lg[:, :E], k, mode, shared=encs[E:], shared_logits=lg[:, E:] if sig else None)
    return got, ref, S


@pytest.mark.parametrize("case", [
    dict(fmt=F.SparseFormat(1, 2, 32), E=8, d=256, f=512, T=100, k=2),
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=257, k=6, gating="softmax_all", shared=2, skew=1.0),
    dict(fmt=F.SparseFormat(1, 2, 32), E=8, d=128, f=256, T=1, k=2),
    dict(fmt=F.SparseFormat(1, 2, 16), E=4, d=256, f=256, T=64, k=2),
    dict(fmt=F.SparseFormat(4, 8, 32), E=4, d=256, f=256, T=64, k=2),
    dict(fmt=F.SparseFormat(8, 16, 32), E=4, d=256, f=256, T=50, k=2),
    dict(fmt=F.SparseFormat(1, 2, 32), E=8, d=256, f=512, T=100, k=2, gate_up="separate"),
    # native (N, 2N, 32) images: interleaved gate/up + down on the in-smem row expansion
    dict(fmt=F.SparseFormat(4, 8, 32), E=4, d=256, f=256, T=300, k=2, transcode="off"),
    dict(fmt=F.SparseFormat(8, 16, 32), E=4, d=256, f=256, T=50, k=2, transcode="off"),
    dict(fmt=F.SparseFormat(4, 8, 32), E=8, d=512, f=640, T=900, k=2, transcode="off", skew=1.0),
    dict(fmt=F.SparseFormat(8, 16, 32), E=16, d=256, f=384, T=257, k=6, gating="softmax_all", shared=2,
         transcode="off"),
    dict(fmt=F.SparseFormat(4, 8, 32), E=8, d=256, f=384, T=7, k=2, transcode="off"),     # decode
    # lane-masked M = 8 slots (separate gate + up, two-weight launch)
    dict(fmt=F.SparseFormat(4, 8, 32), E=4, d=256, f=256, T=300, k=2, transcode="off", gate_up="separate"),
    dict(fmt=F.SparseFormat(2, 2, 32), E=4, d=256, f=512, T=400, k=2),                   # plain 2:4, pair kernels
    # N = M gate + up as two weights of one pair launch (NW = 2: half the gather bytes per MMA)
    dict(fmt=F.SparseFormat(2, 2, 32), E=4, d=512, f=512, T=600, k=2, gate_up="separate"),
    dict(fmt=F.SparseFormat(4, 8, 32), E=4, d=256, f=512, T=500, k=2, gate_up="separate", skew=1.0),
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=57, k=6, gating="softmax_all", shared=2,
         gate_up="separate"),
    # shared experts folded into the grouped launches: top-k fused into the one-block
    # routing (T <= 32), and k + shared = 9 entries per token (Qwen2-like top-8 + 1)
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=20, k=8, gating="softmax_all", shared=1),
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=300, k=8, gating="softmax_all", shared=1),
    # Qwen2-MoE's sigmoid-gated shared expert (reading R15b): a width-4f shared FFN as 4
    # shared experts under one logit per token -- decode (one-block routing) and prefill
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=20, k=4, gating="softmax_all", shared=4,
         shared_gate="sigmoid"),
    dict(fmt=F.SparseFormat(1, 2, 32), E=16, d=256, f=384, T=300, k=8, gating="softmax_all", shared=8,
         shared_gate="sigmoid"),
], ids=lambda c: (f"{c['fmt']}-E{c['E']}-T{c['T']}-{c.get('gate_up', 'auto')}-{c.get('transcode', 'auto')}"
                  f"-sh{c.get('shared', 0)}{c.get('shared_gate', '')}"))
def test_moe_layer_parity(smy, case):
    case = dict(case)
    fmt = case.pop("fmt")
    got, ref, S = _layer_case(smy, fmt, **case)
    check_tol(got, ref, S, "moe layer")


@pytest.mark.parametrize("case", [
    dict(E=4, d=512, f=512, T=512, k=2),                       # tokens/expert >= 64: CTA-pair kernels
    dict(E=8, d=1024, f=768, T=700, k=2, gating="softmax_all"),
    dict(E=2, d=512, f=1024, T=300, k=2, skew=2.0),            # unbalanced experts, ragged tiles
    dict(E=2, d=512, f=512, T=1000, k=2),                      # >= 2 token tiles per expert
    dict(E=4, d=256, f=640, T=400, k=2),                       # interleaved gate/up: 5 m-tiles (odd pair count)
    dict(E=4, d=512, f=512, T=512, k=2, gate_up="separate"),   # two-weight gate/up pair kernel
    dict(E=2, d=512, f=1024, T=300, k=2, skew=2.0, gate_up="separate"),
    dict(E=4, d=512, f=512, T=512, k=2, shared=2),             # shared experts as groups of the pair launches
    dict(E=4, d=512, f=512, T=150, k=2),                       # gate/up: single-CTA NT=128 gather (mid range)
    dict(E=8, d=256, f=768, T=380, k=2, skew=1.0),             # NT=128 gate/up, heavy experts -> 2 token tiles
], ids=lambda c: f"E{c['E']}-d{c['d']}-f{c['f']}-T{c['T']}-{c.get('gate_up', 'auto')}-sh{c.get('shared', 0)}")
def test_moe_layer_prefill_pair_kernels(smy, case):
    case = dict(case)
    got, ref, S = _layer_case(smy, F.SparseFormat(1, 2, 32), **case)
    check_tol(got, ref, S, "moe layer (pair kernels)")


@pytest.mark.parametrize("variant", ["permute", "dense_inter"])
@pytest.mark.parametrize("case", [
    dict(E=4, d=512, f=512, T=512, k=2),                       # CTA-pair kernels
    dict(E=2, d=512, f=1024, T=300, k=2, skew=2.0),            # ragged tiles, unbalanced experts
    dict(E=8, d=256, f=512, T=100, k=2),                       # single-CTA kernels
    dict(E=16, d=256, f=384, T=257, k=6, gating="softmax_all", shared=2, skew=1.0),
], ids=lambda c: f"E{c['E']}-d{c['d']}-f{c['f']}-T{c['T']}-sh{c.get('shared', 0)}")
def test_moe_layer_ablation_variants(smy, variant, case):
    """The breakdown variants (smy_moe_set_variant) compute the same
    layer: the materialised permutation and the token-position intermediate layout
    against the oracle at the layer bar."""
    case = dict(case)
    got, ref, S = _layer_case(smy, F.SparseFormat(1, 2, 32), variant=variant, **case)
    check_tol(got, ref, S, f"moe layer ({variant})")


def test_moe_layer_variant_rejections(smy):
    """A variant applies to the single-GPU interleaved layer only; unknown ids and
    a short scratch are refused without launching."""
    lib = smy.load()
    assert lib.smy_moe_set_variant(7, None, 0) == 3  # SMY_E_CONFIG
    assert lib.smy_moe_set_variant(1, None, 0) != 0  # needs scratch
    assert lib.smy_moe_set_variant(0, None, 0) == 0


@pytest.mark.parametrize("T", [1, 100, 600])
def test_moe_layer_bf16_output(smy, T):
    """cfg.out_dtype = bf16 (reading R13: optional bf16 layer output, compared
    after emulated rounding): fp32 accumulation, one RNE rounding -- against the
    oracle's output rounded to bf16: rel Frobenius <= 1e-3 and every element
    within one bf16 ulp plus the north-star per-element bound."""
    fmt = F.SparseFormat(1, 2, 32)
    E, d, f, k = 8, 256, 512, 2
    encs, sws = [], []
    for e in range(E):
        te, ts = [], []
        for i in range(3):
            r, c = (f, d) if i < 2 else (d, f)
            w = synth.weight_bf16(synth.weight_seed(e, i), r, c)
            te.append(F.encode(F.prune(w, fmt), fmt))
            ts.append(smy.compress(dev16(w), gpu_format(fmt))[0])
        encs.append(tuple(te))
        sws.append(tuple(ts))
    x = synth.activations_bf16(synth.SEED_X, T, d)
    lg = synth.router_logits(synth.SEED_LOGITS, T, E)
    layer = smy.MoELayer(smy.MoEConfig(E, k, d, f, out_dtype="bf16"), sws, max_tokens=T)
    out = layer(dev16(x), torch.from_numpy(lg).cuda())
    assert out.dtype == torch.bfloat16 and tuple(out.shape) == (T, d)
    got = bf16.to_f64(host16(out.view(torch.int16)))
    ref64, S = moe.moe_layer(encs, x, lg, k)
    ref = bf16.to_f64(bf16.from_f64(ref64))
    assert OS.rel_fro(got - ref, ref) <= REL_FRO
    bad = np.abs(got - ref) > np.maximum(bf16_ulp(ref), bf16_ulp(got)) + ELEM * S + 1e-30
    assert not bad.any(), np.argwhere(bad)[:3]


def test_moe_layer_all_tokens_one_expert(smy):
    fmt = F.SparseFormat(1, 2, 32)
    got, ref, S = _layer_case(smy, fmt, E=4, d=128, f=256, T=200, k=1, skew=50.0)
    check_tol(got, ref, S, "hot expert")


# ------------------------------------------------ full size, bench launch configuration

def _prune_rows(w_bits, fmt, chunk=512):
    """oracle prune, row-chunked (pruning acts on M-row groups independently)."""
    return np.concatenate([F.prune(w_bits[i:i + chunk], fmt) for i in range(0, w_bits.shape[0], chunk)])


def _tile_positions(n):
    """positions in an expert's SEL that fall in its first, a middle and its last
    (ragged) token tile: the first two, the middle two and the last two rows"""
    return sorted({p for p in (0, 1, n // 2, n // 2 + 1, n - 2, n - 1) if 0 <= p < n})


@pytest.mark.parametrize("model,T,NS", [("mixtral", 4096, 0), ("mixtral", 64, 0), ("deepseek", 4096, 0),
                                        ("deepseek", 4096, 2), ("deepseek", 64, 2), ("qwen2", 4096, 0),
                                        ("qwen2", 64, 0)])
def test_moe_layer_full_size_sampled(smy, model, T, NS):
    """The bench's workloads themselves -- Mixtral-8x7B / DeepSeek-MoE-16B /
    Qwen2-57B-A14B layers at T=4096 (interleaved gate/up + stream-K down on CTA
    pairs) and T=64 decode points (single-CTA kernels), built by
    bench.build_layer -- checked against the fp64 oracle on samples that cover
    every part of the tile schedule: for 4 routed experts spread over the expert
    range (+ every shared expert), the tokens at the first two, middle two and
    last two positions of the expert's SEL (its first, a middle and its last,
    ragged token tile -- and so the stream-K pieces of the down launch).
      * gate/up intermediate: the layer's own compact bf16 buffer
        (MoELayer.view) on 32 sampled channel pairs of those (expert, token)
        rows, at the north-star bar (check_silu_mul);
      * layer output: those tokens x 24 sampled output row pairs.
    The oracle regenerates the weights it needs by index (counter-based
    generator) and prunes them itself.  NS > 0: the layer also runs NS shared
    experts (bench.py --shared; every token, weight 1), drawn like routed experts
    E, E+1, ..."""
    import bench
    d, f, E, k, gating = bench.MODELS[model]
    fmt = F.SparseFormat(1, 2, 32)
    dev = torch.device("cuda")
    shared = bench.build_layer(smy, model, dev, experts=range(E, E + NS)) if NS else ()
    layer = smy.MoELayer(smy.MoEConfig(E, k, d, f, NS, gating, smy.Format(1, 2, 32)),
                         bench.build_layer(smy, model, dev), shared=shared, max_tokens=T, device=dev)
    x = torch.empty(T, d, dtype=torch.int16, device=dev)
    smy.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    lg = torch.empty(T, E, dtype=torch.float32, device=dev)
    smy.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    out = layer(x, lg).cpu().numpy().astype(np.float64)
    v = layer.view(T)
    offsets = v["offsets"].cpu().numpy()
    sel_all = v["sel"].cpu().numpy()
    inter = host16(v["inter"])
    xh, lgh = host16(x), lg.cpu().numpy()
    del layer, shared, v
    torch.cuda.empty_cache()

    ids, gw = moe.route(lgh, k, moe.SOFTMAX_ALL if gating == "softmax_all" else moe.RENORM_TOPK)
    _, r_off, r_sel, _ = moe.compact(ids, gw, E)
    assert np.array_equal(offsets[:E + 1], r_off) and np.array_equal(sel_all[:r_off[E]], r_sel)

    def dense(seed, rows, cols, idx0=0):
        t = torch.empty(rows, cols, dtype=torch.int16, device=dev)
        smy.synth_fill(t, seed, synth.DIST_UNIFORM, float(synth.uniform_scale(np.sqrt(3.0 / cols))), idx0=idx0)
        return host16(t)

    def pruned_rows(seed, cols, groups):
        """rows 2g, 2g+1 of a weight with `cols` columns, pruned by the oracle"""
        w = np.concatenate([dense(seed, 2, cols, idx0=int(2 * g) * cols) for g in groups])
        return bf16.to_f64(F.prune(w, fmt))

    rng = np.random.default_rng(3)
    routed = sorted({int(e) for e in np.linspace(0, E - 1, 4).round()})
    picks = {}                                          # expert -> [(row in the compact buffer, token)]
    for e in routed + list(range(E, E + NS)):
        o0, n = int(offsets[e]), int(offsets[e + 1] - offsets[e])
        picks[e] = [(o0 + p, int(sel_all[o0 + p])) for p in _tile_positions(n)]
    assert sum(len(p) for p in picks.values()) >= 4

    # ---- gate/up intermediate of those (expert, token) rows, sampled channel pairs
    cgroups = np.sort(rng.choice(f // 2, 32, replace=False))
    chan = np.sort(np.concatenate([2 * cgroups, 2 * cgroups + 1]))
    for e, pk in picks.items():
        if not pk:
            continue
        xs = bf16.to_f64(xh[[t for _, t in pk]])
        wg = pruned_rows(synth.weight_seed(e, 0), d, cgroups)
        wu = pruned_rows(synth.weight_seed(e, 1), d, cgroups)
        got = bf16.to_f64(inter[np.ix_([r for r, _ in pk], chan)])
        check_silu_mul(got, xs @ wg.T, xs @ wu.T, np.abs(xs) @ np.abs(wg).T, np.abs(xs) @ np.abs(wu).T,
                       f"{model} T={T} gate/up intermediate, expert {e}, SEL rows {[r for r, _ in pk]}")

    # ---- layer output of those tokens
    toks = np.array(sorted({t for pk in picks.values() for _, t in pk}))
    xs = bf16.to_f64(xh[toks])
    groups = np.sort(rng.choice(d // 2, 24, replace=False))
    orow = np.sort(np.concatenate([2 * groups, 2 * groups + 1]))
    ref = np.zeros((len(toks), len(orow)))
    S = np.zeros_like(ref)
    need = sorted({int(e) for t in toks for e in ids[t]}) + list(range(E, E + NS))
    for e in need:
        rows = [i for i, t in enumerate(toks) if e >= E or e in ids[t]]
        wg = bf16.to_f64(_prune_rows(dense(synth.weight_seed(e, 0), f, d), fmt))
        wu = bf16.to_f64(_prune_rows(dense(synth.weight_seed(e, 1), f, d), fmt))
        xe = xs[rows]
        a = bf16.to_f64(OS.silu_mul_bf16(xe @ wg.T, xe @ wu.T))             # [rows x f] bf16 intermediate
        del wg, wu
        wd = pruned_rows(synth.weight_seed(e, 2), f, groups)                 # rows orow
        g_e = (np.array([gw[toks[i]][list(ids[toks[i]]).index(e)] for i in rows])[:, None] if e < E
               else np.ones((len(rows), 1)))                                 # shared expert: weight 1
        ref[rows] += g_e * (a @ wd.T)
        S[rows] += np.abs(g_e) * (np.abs(a) @ np.abs(wd).T)
    check_tol(out[np.ix_(toks, orow)], ref, S,
              f"{model} T={T} layer (+{NS} shared), {len(toks)} tokens from the first/middle/last tiles of "
              f"experts {sorted(picks)}")
