"""CPU-only checks of the C ABI boundary: the library builds/loads, exports every
symbol include/samoyeds.h declares, and its host-side queries/validation work
without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "samoyeds.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^SMY_API\s+[\w\s\*]+?\b(\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_10725_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2503_10725_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("samoyeds_compress", "samoyeds_ssmm", "samoyeds_moe_layer", "samoyeds_route"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2503_10725_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"binding lacks {name}"


def test_layout_query_closed_forms(lib):
    from paper_2503_10725_b200 import Format, weight_layout
    L = weight_layout(14336, 4096, Format(1, 2, 32))
    assert L["values"] == 7168 * 2048 * 2
    assert L["codes"] == 7168 * 4096 // 8
    assert L["indices"] == 7168 * 4096 // 32
    assert L["m_tiles"] == 56 and L["k_stages"] == 32 and L["planes"] == 1 and L["rep"] == 1
    total = L["values"] + L["codes"] + L["indices"]
    assert total / (14336 * 4096) == 0.578125
    L16 = weight_layout(128, 256, Format(1, 2, 16))
    assert L16["rep"] == 2 and L16["k_stages"] == 4
    assert weight_layout(1408, 2048, Format(2, 2, 32))["planes"] == 0
    assert weight_layout(512, 512, Format(8, 16, 32))["planes"] == 4


def test_host_validation_without_gpu(lib):
    from paper_2503_10725_b200._lib import smy_wdesc, smy_format, smy_wlayout
    lay = smy_wlayout()
    for rows, cols, f, want in ((129, 256, (1, 2, 32), 2), (128, 200, (1, 2, 32), 2), (128, 256, (3, 2, 32), 3),
                                (128, 256, (1, 2, 8), 3), (128, 256, (2, 4, 16), 3)):
        d = smy_wdesc(rows, cols, smy_format(*f))
        assert lib.smy_weight_layout(C.byref(d), C.byref(lay)) == want
    assert lib.smy_weight_layout(None, C.byref(lay)) == 1
    assert lib.smy_status_str(4) == b"SMY_E_PATTERN"
    b = C.c_size_t()
    assert lib.smy_route_workspace_bytes(4096, 64, C.byref(b)) == 0 and b.value > 0


def test_moe_layer_shared_expert_limits_without_gpu(lib):
    """samoyeds_moe_layer validates on the host, before any device work: shared
    experts become extra groups (E + shared <= 128) and extra routing entries per
    token (top_k + shared <= 16) -- include/samoyeds.h."""
    from paper_2503_10725_b200 import MoEConfig, Format
    from paper_2503_10725_b200._lib import smy_weight
    ws = (smy_weight * 2)()
    dummy = (C.c_uint8 * 16)()
    p = C.cast(dummy, C.c_void_p)
    for E, k, ns in ((127, 2, 2), (64, 8, 9)):
        cfg = MoEConfig(E, k, 256, 256, ns, fmt=Format(1, 2, 32)).c()
        st = lib.samoyeds_moe_layer(C.byref(cfg), ws, ws, p, p, 16, p, p, 16, None, None)
        assert st == 3, (E, k, ns, st)   # SMY_E_CONFIG


def test_moe_workspace_query(lib):
    from paper_2503_10725_b200 import MoEConfig, Format
    from paper_2503_10725_b200._lib import check
    cfg = MoEConfig(8, 2, 4096, 14336, fmt=Format(1, 2, 32)).c()
    b = C.c_size_t()
    check(lib.smy_moe_workspace_bytes(C.byref(cfg), 4096, C.byref(b)), "ws")
    assert b.value >= 4096 * 2 * 14336 * 2                         # the bf16 intermediate


def _fake_weight(rows, cols, fmt, addr):
    """an smy_weight whose (never dereferenced) device pointers are `addr`"""
    from paper_2503_10725_b200._lib import smy_format, smy_wdesc, smy_weight
    p = C.c_void_p(addr)
    return smy_weight(smy_wdesc(rows, cols, smy_format(*fmt)), p, p, p, p)


def test_ssmm_scatter_alignment_rejected_without_gpu(lib):
    """SCATTER_ADD reduces 16 B per lane pair: ldo % 4, a 16-B aligned out and
    rows % 4 are checked on the host, before the arch check."""
    w = _fake_weight(256, 256, (1, 2, 32), 0x10000)
    p = C.c_void_p(0x20000)
    # ldo = 258 (even, >= rows, not % 4)
    assert lib.samoyeds_ssmm(C.byref(w), None, p, 256, 64, p, 16, None, 2, p, 258, 0, None) == 2
    # out 8-B aligned only
    assert lib.samoyeds_ssmm(C.byref(w), None, p, 256, 64, p, 16, None, 2, C.c_void_p(0x20008), 256, 0, None) == 2
    # rows = 258 (% M == 0, not % 4)
    w2 = _fake_weight(258, 256, (1, 2, 32), 0x10000)
    assert lib.samoyeds_ssmm(C.byref(w2), None, p, 256, 64, p, 16, None, 2, p, 260, 0, None) == 2


def test_interleave_rejects_formats_without_16_row_blocks(lib):
    """samoyeds_interleave_gate_up moves blocks of 16 compressed rows: weights with
    R = rows * N / M not a multiple of 16 are rejected (the oracle's
    interleave_gate_up requires rows % (16 M / N))."""
    for fmt, rows, want in (((1, 4, 32), 32, 2), ((1, 8, 32), 64, 2), ((1, 2, 32), 48, 2)):
        g = _fake_weight(rows, 256, fmt, 0x10000)
        u = _fake_weight(rows, 256, fmt, 0x20000)
        gu = _fake_weight(2 * rows, 256, fmt, 0x30000)
        assert lib.samoyeds_interleave_gate_up(C.byref(g), C.byref(u), C.byref(gu), None) == want, fmt


def test_moe_layer_rejects_unknown_gating_and_misaligned_out(lib):
    from paper_2503_10725_b200 import MoEConfig, Format
    from paper_2503_10725_b200._lib import smy_weight
    ws = (smy_weight * 24)()
    p = C.c_void_p(0x10000)
    cfg = MoEConfig(8, 2, 256, 256, fmt=Format(1, 2, 32)).c()
    cfg.gating = 7
    assert lib.samoyeds_moe_layer(C.byref(cfg), ws, None, p, p, 16, p, p, 16, None, None) == 3
    cfg.gating = 0
    assert lib.samoyeds_moe_layer(C.byref(cfg), ws, None, p, p, 16, C.c_void_p(0x10004), p, 16, None, None) == 2
    # samoyeds_moe_experts has no shared experts
    cfg.num_shared = 1
    assert lib.samoyeds_moe_experts(C.byref(cfg), ws, p, 16, p, p, p, p, 16, None) == 3


@pytest.mark.parametrize("model,fmt,T,gu_expect,dn_expect", [
    # prefill: gate/up m-tile-paired on the CTA pair (NT=112), down on the pair at NT=224
    ("mixtral", (1, 2, 32), 4096, "ssmm_pair_kernel<112, 2, 2, 1>", "ssmm_pair_kernel<224, 1, 2, 0>"),
    ("deepseek", (1, 2, 32), 4096, "ssmm_pair_kernel<112, 2, 2, 1>", "ssmm_pair_kernel<224, 1, 2, 0>"),
    # mid range: <= 128-token gate/up tiles stay single-CTA, the down goes to the pair
    ("mixtral", (1, 2, 32), 256, "ssmm_kernel<128, 1, 2, 1>", "ssmm_pair_kernel<128, 1, 2, 0>"),
    # decode: single-CTA kernels with narrow token tiles
    ("mixtral", (1, 2, 32), 64, "ssmm_kernel<32, 1, 2, 1>", "ssmm_kernel<32, 1, 2, 1>"),
    ("qwen2", (1, 2, 32), 1, "ssmm_kernel<16, 1, 2, 1>", "ssmm_kernel<16, 1, 2, 1>"),
    # N = M (and N>1 formats transcoded to it): gate + up and the m-tile-paired down at NT=224
    ("mixtral", (4, 8, 32), 4096, "ssmm_pair_kernel<224, 2, 1, 1>", "ssmm_pair_kernel<224, 2, 1, 1>"),
    ("mixtral", (2, 2, 32), 4096, "ssmm_pair_kernel<224, 2, 1, 1>", "ssmm_pair_kernel<224, 2, 1, 1>"),
    # native (N, 2N, 32) images (transcode "off"): the in-smem row expansion (XP = 1)
    ("mixtral", (4, 8, 32, "off"), 64, "ssmm_kernel<32, 1, 2, 1, 1>", "ssmm_kernel<32, 1, 2, 1, 1>"),
    ("deepseek", (8, 16, 32, "off"), 4096, "ssmm_kernel<128, 1, 2, 1, 1>", "ssmm_kernel<128, 1, 2, 1, 1>"),
])
def test_kernel_selection_rules(lib, model, fmt, T, gu_expect, dn_expect):
    """The launch decisions of samoyeds_moe_layer (tile width, CTA pair vs single CTA,
    m-tile pairing) as smy_moe_kernel_names reports them -- host-only."""
    import bench
    from paper_2503_10725_b200 import api
    d, f, E, k, gating = bench.MODELS[model]
    tc = fmt[3] if len(fmt) > 3 else "auto"
    cfg = api.MoEConfig(E, k, d, f, 0, gating, api.Format(*fmt[:3]), transcode=tc).kernel_config().c()
    gu, dn = C.create_string_buffer(96), C.create_string_buffer(96)
    assert lib.smy_moe_kernel_names(C.byref(cfg), T, gu, dn, 96) == 0
    assert (gu.value.decode(), dn.value.decode()) == (gu_expect, dn_expect)
