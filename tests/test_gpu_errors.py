"""GPU checks of the C ABI's data-dependent error paths and input edge cases
(include/samoyeds.h): corrupt encodings (SMY_E_CORRUPT), SEL validation
(SMY_E_SELECTION), NaN router logits, and routing keys outside [0, E)."""
import numpy as np
import pytest
import torch

import synth
from oracle import fmt as F, moe, ssmm as OS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def smy():
    import paper_2503_10725_b200 as P
    P.load()
    return P


def dev16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda()


@pytest.mark.parametrize("fmt", [F.SparseFormat(1, 2, 32), F.SparseFormat(4, 8, 32)], ids=str)
def test_decompress_reports_corrupt_encodings(smy, fmt):
    """A sub-row index >= M, indices out of order, or a 4-group whose two codes are
    not increasing -> SMY_E_CORRUPT (6) in the status word; intact -> 0 (the
    invariants of the oracle's fmt.validate)."""
    w = synth.weight_bf16(91, 256, 256)
    sw, _ = smy.compress(dev16(w), smy.Format(fmt.n, fmt.m, fmt.v))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    dense = smy.decompress(sw, status=st)
    assert int(st.item()) == 0
    assert np.array_equal(dense.cpu().numpy().view(np.uint16), F.prune(w, fmt))
    good_idx, good_codes = sw.indices.clone(), sw.codes.clone()
    cases = {"index >= M": lambda: sw.indices.__setitem__(0, fmt.m),
             "codes not increasing": lambda: sw.codes.__setitem__(0, 0x00)}   # (0,0) for the first 4-group
    if fmt.n > 1:
        J = 256 // fmt.v
        cases["indices not increasing"] = lambda: (sw.indices.__setitem__(0, 1), sw.indices.__setitem__(J, 0))
    for name, corrupt in cases.items():
        sw.indices.copy_(good_idx)
        sw.codes.copy_(good_codes)
        corrupt()
        st.zero_()
        smy.decompress(sw, status=st)
        torch.cuda.synchronize()
        assert int(st.item()) == 6, name


def test_validate_sel(smy):
    ok = torch.tensor([0, 3, 4, 9, 63], dtype=torch.int32, device="cuda")
    assert int(smy.validate_sel(ok, 64).item()) == 0
    assert int(smy.validate_sel(ok[:0], 64).item()) == 0
    for bad in ([0, 3, 3, 9], [0, 5, 4], [-1, 2], [1, 64]):
        t = torch.tensor(bad, dtype=torch.int32, device="cuda")
        assert int(smy.validate_sel(t, 64).item()) == 5, bad


def test_route_nan_logits(smy):
    """A NaN logit ranks as -inf (reading R10b): ids bit-exact and weights as the
    oracle's, for both gating modes."""
    lg = synth.router_logits(synth.SEED_LOGITS, 300, 16)
    rng = np.random.default_rng(5)
    lg[rng.random(lg.shape) < 0.2] = np.nan
    lg[7, :] = np.nan
    lg[7, 3] = 1.0                                   # one finite logit in the row
    for gating, mode in (("renorm_topk", moe.RENORM_TOPK), ("softmax_all", moe.SOFTMAX_ALL)):
        ids, w, counts, offsets, sel, gw = smy.route(torch.from_numpy(lg).cuda(), 4, gating)
        rid, rw = moe.route(lg, 4, mode)
        assert np.array_equal(ids.cpu().numpy(), rid)
        assert np.allclose(w.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)
        rc, ro, rs, _ = moe.compact(rid, rw, 16)
        assert np.array_equal(sel.cpu().numpy(), rs)


def test_moe_experts_ignores_keys_outside_range(smy):
    """samoyeds_moe_experts: routing keys >= E (like negative ones) are no entry --
    no out-of-bounds mask write, the rows get only their valid experts."""
    fmt = F.SparseFormat(1, 2, 32)
    E, k, d, f, R = 4, 2, 128, 256, 40
    encs, sws = [], []
    for e in range(E):
        te, ts = [], []
        for i in range(3):
            r, c = (f, d) if i < 2 else (d, f)
            w = synth.weight_bf16(synth.weight_seed(e, i), r, c)
            te.append(F.encode(F.prune(w, fmt), fmt))
            ts.append(smy.compress(dev16(w), smy.Format(1, 2, 32))[0])
        encs.append(tuple(te))
        sws.append(tuple(ts))
    x = synth.activations_bf16(3, R, d)
    rng = np.random.default_rng(1)
    keys = rng.integers(0, E, (R, k)).astype(np.int32)
    keys[:, 1] = np.where(keys[:, 1] == keys[:, 0], (keys[:, 0] + 1) % E, keys[:, 1])
    vals = rng.random((R, k)).astype(np.float32)
    bad = keys.copy()
    bad[::3, 1] = E + 5                              # outside [0, E)
    bad[1::3, 1] = 1 << 20
    layer = smy.MoEExperts(smy.MoEConfig(E, k, d, f), sws, max_rows=R)
    got = layer(dev16(x), torch.from_numpy(bad).cuda(), torch.from_numpy(vals).cuda()).cpu().numpy()
    ref = np.zeros((R, d))
    S = np.zeros((R, d))
    for e in range(E):
        rows = [r for r in range(R) for j in range(k) if bad[r, j] == e]
        if not rows:
            continue
        y, _, Se = moe.expert_ffn(*encs[e], x, np.array(rows))
        for i, r in enumerate(rows):
            g = vals[r][list(bad[r]).index(e)]
            ref[r] += g * y[i]
            S[r] += abs(g) * Se[i]
    assert OS.rel_fro(got - ref, ref) <= 1e-3
    assert (np.abs(got - ref) <= 1e-2 * S + 1e-30).all()
