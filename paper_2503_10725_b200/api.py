"""Python API over the C ABI (include/samoyeds.h) -- argument marshalling only.

PyTorch provides device memory and streams; every step of the path runs in
libsamoyeds.so kernels.  Names follow the C ABI and the paper's notation.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import check, smy_format, smy_moe_config, smy_wdesc, smy_weight, smy_wlayout

EPI = {"compact": 0, "silu_mul": 1, "scatter_add": 2, "silu_mul_interleaved": 3}
GATE_UP = {"separate": 0, "interleaved": 1}
GATING = {"renorm_topk": 0, "softmax_all": 1}
SHARED_GATE = {"none": 0, "sigmoid": 0x10}   # SMY_GATE_SHARED_SIGMOID
PRUNE_MAGNITUDE = 1
ASSUME_PRUNED = 2


def _stream(stream=None) -> C.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (no CPU path)")
    return C.c_void_p(t.data_ptr())


@dataclass(frozen=True)
class Format:
    """(N, M, V) vector-wise sparsity on top of 2:4."""
    n: int = 1
    m: int = 2
    v: int = 32

    def c(self) -> smy_format:
        return smy_format(self.n, self.m, self.v)


def weight_layout(rows: int, cols: int, fmt: Format) -> dict:
    lib = _lib.load()
    d = smy_wdesc(rows, cols, fmt.c())
    lay = smy_wlayout()
    check(lib.smy_weight_layout(C.byref(d), C.byref(lay)), "smy_weight_layout")
    return {f: getattr(lay, f) for f, _ in smy_wlayout._fields_}


class SparseWeight:
    """An encoded weight: canonical (values, codes, indices) + device image."""

    def __init__(self, rows: int, cols: int, fmt: Format, device=None, image: Optional[torch.Tensor] = None):
        """`image`: optional caller-provided uint8 view of layout["image"] bytes
        (e.g. a slice of one block holding every expert's image)."""
        self.rows, self.cols, self.fmt = rows, cols, fmt
        self.layout = weight_layout(rows, cols, fmt)
        dev = device or torch.device("cuda")
        L = self.layout
        self.values = torch.empty(L["values"] // 2, dtype=torch.int16, device=dev)
        self.codes = torch.empty(L["codes"], dtype=torch.uint8, device=dev)
        self.indices = torch.empty(L["indices"], dtype=torch.uint8, device=dev)
        if image is not None and (image.dtype != torch.uint8 or image.numel() != L["image"] or
                                  not image.is_contiguous()):
            raise ValueError("image must be a contiguous uint8 tensor of layout['image'] bytes")
        self.image = torch.empty(L["image"], dtype=torch.uint8, device=dev) if image is None else image

    def c(self) -> smy_weight:
        return smy_weight(smy_wdesc(self.rows, self.cols, self.fmt.c()), _ptr(self.values), _ptr(self.codes),
                          _ptr(self.indices), _ptr(self.image))

    @property
    def nbytes_canonical(self) -> int:
        return self.values.numel() * 2 + self.codes.numel() + self.indices.numel()

    def drop_canonical(self) -> None:
        """Free the canonical copy; the SSMM only reads the device image."""
        self.values = self.codes = self.indices = None


def compress(w: torch.Tensor, fmt: Format, prune: bool = True, stream=None):
    """samoyeds_compress: w is a CUDA bf16 (or int16 bit-pattern) [rows x cols]
    tensor.  Returns (SparseWeight, status tensor int32[1])."""
    lib = _lib.load()
    if w.dtype == torch.bfloat16:
        w = w.view(torch.int16)
    assert w.dtype == torch.int16 and w.dim() == 2 and w.stride(1) == 1
    rows, cols = w.shape
    sw = SparseWeight(rows, cols, fmt, w.device)
    status = torch.zeros(1, dtype=torch.int32, device=w.device)
    d = smy_wdesc(rows, cols, fmt.c())
    cw = sw.c()
    check(lib.samoyeds_compress(C.byref(d), _ptr(w), w.stride(0), PRUNE_MAGNITUDE if prune else ASSUME_PRUNED,
                                C.byref(cw), _ptr(status), _stream(stream)), "samoyeds_compress")
    return sw, status


def decompress(w: SparseWeight, stream=None, status: Optional[torch.Tensor] = None) -> torch.Tensor:
    """samoyeds_decompress: the dense bf16 [rows x cols] (int16 bit patterns) weight.
    status: optional zeroed int32[1] CUDA tensor; receives SMY_E_CORRUPT (6) if the
    canonical arrays violate the decoding invariants."""
    lib = _lib.load()
    if w.values is None:
        raise ValueError("decompress needs the canonical arrays (drop_canonical() was called)")
    out = torch.empty(w.rows, w.cols, dtype=torch.int16, device=w.image.device)
    cw = w.c()
    check(lib.samoyeds_decompress(C.byref(cw), _ptr(out), out.stride(0), _ptr(status) if status is not None else None,
                                  _stream(stream)), "samoyeds_decompress")
    return out


def validate_sel(sel: torch.Tensor, x_rows: int, stream=None) -> torch.Tensor:
    """samoyeds_validate_sel: int32[1] status tensor (0, or SMY_E_SELECTION = 5 if
    sel is not strictly increasing within [0, x_rows)); asynchronous."""
    lib = _lib.load()
    status = torch.zeros(1, dtype=torch.int32, device=sel.device)
    check(lib.samoyeds_validate_sel(_ptr(sel), sel.numel(), x_rows, _ptr(status), _stream(stream)),
          "samoyeds_validate_sel")
    return status


def transcode_24(w: SparseWeight, stream=None) -> SparseWeight:
    """The same weight re-encoded as plain 2:4, format (2,2,32) (N = M: every
    sub-row kept, zero sub-rows stored as zeros): decompress + compress
    (ASSUME_PRUNED).  Twice the image bytes of an N/M = 1/2 format, but it runs
    on the fast N = M kernels -- how N>1 and V=16 formats reach speed."""
    dense = decompress(w, stream)
    out, _ = compress(dense, Format(2, 2, 32), prune=False, stream=stream)
    return out


def interleave_gate_up(gate: SparseWeight, up: SparseWeight, stream=None,
                       image: Optional[torch.Tensor] = None) -> SparseWeight:
    """samoyeds_interleave_gate_up: the [2f x d] gate/up weight whose 128-row
    blocks alternate gate and up rows (reading R20).  Needs the
    canonical arrays of both inputs.  `image`: optional preallocated image view."""
    lib = _lib.load()
    if gate.values is None or up.values is None:
        raise ValueError("interleave_gate_up needs the canonical arrays (drop_canonical() was called)")
    gu = SparseWeight(2 * gate.rows, gate.cols, gate.fmt, gate.image.device, image=image)
    cg, cu, cgu = gate.c(), up.c(), gu.c()
    check(lib.samoyeds_interleave_gate_up(C.byref(cg), C.byref(cu), C.byref(cgu), _stream(stream)),
          "samoyeds_interleave_gate_up")
    return gu


def ssmm(w: SparseWeight, x: torch.Tensor, sel: torch.Tensor, epi: str = "compact",
         w2: Optional[SparseWeight] = None, scale: Optional[torch.Tensor] = None,
         out: Optional[torch.Tensor] = None, out_dtype=torch.float32, stream=None) -> torch.Tensor:
    """samoyeds_ssmm.  x: CUDA bf16 [x_rows x cols] token-major; sel: int32
    [n_sel].  compact/silu_mul return [n_sel x rows]; scatter_add accumulates
    into ``out`` [x_rows x rows] (fp32) and returns it."""
    lib = _lib.load()
    n_sel = sel.numel()
    if out is None:
        if epi == "scatter_add":
            raise ValueError("scatter_add needs an output tensor")
        dt = torch.bfloat16 if epi.startswith("silu_mul") else out_dtype
        cols = w.rows // 2 if epi == "silu_mul_interleaved" else w.rows
        out = torch.empty(n_sel, cols, dtype=dt, device=x.device)
    odt = 1 if out.dtype == torch.bfloat16 else 0
    xb = x.view(torch.int16) if x.dtype == torch.bfloat16 else x
    cw = w.c()
    cw2 = w2.c() if w2 is not None else None
    check(lib.samoyeds_ssmm(C.byref(cw), C.byref(cw2) if cw2 is not None else None, _ptr(xb), xb.stride(0),
                            xb.shape[0], _ptr(sel), n_sel, _ptr(scale), EPI[epi], _ptr(out), out.stride(0), odt,
                            _stream(stream)), "samoyeds_ssmm")
    return out


def route(logits: torch.Tensor, k: int, gating: str = "renorm_topk", stream=None):
    """samoyeds_route: top-k + gate weights + per-expert selection arrays."""
    lib = _lib.load()
    T, E = logits.shape
    dev = logits.device
    ws_bytes = C.c_size_t()
    check(lib.smy_route_workspace_bytes(T, E, C.byref(ws_bytes)), "smy_route_workspace_bytes")
    ws = torch.empty(max(ws_bytes.value, 1), dtype=torch.uint8, device=dev)
    ids = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    offsets = torch.empty(E + 1, dtype=torch.int32, device=dev)
    sel = torch.empty(max(T * k, 1), dtype=torch.int32, device=dev)
    gw = torch.empty(max(T * k, 1), dtype=torch.float32, device=dev)
    check(lib.samoyeds_route(_ptr(logits), T, E, k, GATING[gating], _ptr(ids), _ptr(w), _ptr(counts),
                             _ptr(offsets), _ptr(sel), _ptr(gw), _ptr(ws), ws.numel(), _stream(stream)),
          "samoyeds_route")
    return ids, w, counts, offsets, sel[:T * k], gw[:T * k]


@dataclass
class MoEConfig:
    num_experts: int
    top_k: int
    hidden: int
    ffn: int
    num_shared: int = 0
    gating: str = "renorm_topk"
    fmt: Format = Format()
    # "auto": the interleaved gate/up weight (one SSMM, reading R20) whenever the
    # format allows it -- (1,2,V) or N = M, V % 32 == 0 -- else separate gate and up
    gate_up: str = "auto"
    # "auto": formats without fast kernels (N>1 with N<M, V=16) are re-encoded as
    # plain 2:4 (2,2,32) when a layer is built (transcode_24); "off": keep them
    transcode: str = "auto"
    # layer output dtype: "f32" (default) or "bf16" (fp32 accumulation in the
    # workspace, one RNE rounding at the end; single-GPU layer)
    out_dtype: str = "f32"
    # shared experts' weight: "none" = 1 (reading R15); "sigmoid" = sigmoid of a
    # per-token shared-gate logit, taken from logits[:, num_experts + s] (the
    # logits then have num_experts + num_shared columns; Qwen2-MoE, reading R15b)
    shared_gate: str = "none"

    def fast_format(self) -> bool:
        f = self.fmt
        return f.v % 32 == 0 and ((f.n == 1 and f.m == 2) or f.n == f.m)

    def resolved_gate_up(self) -> str:
        if self.gate_up != "auto":
            return self.gate_up
        # (1,2,V): the interleaved weight (one SSMM, two lane-masked slots); N = M:
        # gate and up as the two weights of one launch (two accumulators per token
        # stage, half the SEL-gather bytes per MMA of the interleaved one-slot
        # kernel: Mixtral (2,2,32) gate/up 2.04 -> 1.08 ms, profiles/r2_nm_formats.md)
        # (N,2N,V), N > 1, kept native (transcode "off"): the interleaved weight too --
        # every one-weight SSMM of these formats runs the in-smem row expansion (§7.5)
        f = self.fmt
        ok = f.v % 32 == 0 and f.m == 2 * f.n and self.ffn % 128 == 0
        return "interleaved" if ok else "separate"

    def kernel_config(self) -> "MoEConfig":
        """The configuration the layer's kernels run on (after transcoding)."""
        if self.transcode == "auto" and not self.fast_format():
            return MoEConfig(self.num_experts, self.top_k, self.hidden, self.ffn, self.num_shared, self.gating,
                             Format(2, 2, 32), self.gate_up, "off", self.out_dtype, self.shared_gate)
        return self

    def c(self) -> smy_moe_config:
        return smy_moe_config(self.num_experts, self.top_k, self.hidden, self.ffn, self.num_shared,
                              GATING[self.gating] | SHARED_GATE[self.shared_gate], self.fmt.c(),
                              GATE_UP[self.resolved_gate_up()],
                              {"f32": 0, "bf16": 1}[self.out_dtype])


def _weight_array(triples: Sequence[Sequence[Optional[SparseWeight]]]):
    flat = [w for t in triples for w in t]
    arr = (smy_weight * len(flat))(*[w.c() if w is not None else smy_weight() for w in flat])
    return arr


def prepare_experts(cfg: MoEConfig, triples, stream=None):
    """(gate, up, down) triples -> the layout cfg.kernel_config().c() announces:
    transcoded to plain 2:4 if the format has no fast kernels, then unchanged for
    "separate", (gu, None, down) with gu = interleave_gate_up(gate, up) for
    "interleaved"."""
    kc = cfg.kernel_config()
    if kc is not cfg and triples and all(t[1] is not None for t in triples) and triples[0][0].fmt != kc.fmt:
        triples = [tuple(transcode_24(w, stream) for w in t) for t in triples]
    cfg = kc
    if cfg.resolved_gate_up() == "separate":
        return [tuple(t) for t in triples]
    if not triples or all(t[1] is None for t in triples):   # already (gu, None, down)
        return [tuple(t) for t in triples]
    # one block for all experts' images: a grouped CTA-pair launch addresses them
    # through a single tensor map (include/samoyeds.h, samoyeds_moe_layer)
    g0 = triples[0][0]
    nb = weight_layout(2 * g0.rows, g0.cols, g0.fmt)["image"]
    block = torch.empty(len(triples) * nb, dtype=torch.uint8, device=g0.image.device)
    return [(interleave_gate_up(g, u, stream, image=block[i * nb:(i + 1) * nb]), None, d)
            for i, (g, u, d) in enumerate(triples)]


class EPComm:
    """smy_ep_comm: the library-owned NCCL communicator of expert parallelism.
    Rank 0 draws the NCCL unique id (smy_ep_unique_id); it is broadcast over the
    torch process group `group`, then every rank joins (smy_ep_comm_create)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        lib = _lib.load()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            check(lib.smy_ep_unique_id(uid), "smy_ep_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        self.handle = C.c_void_p()
        check(lib.smy_ep_comm_create(uid, self.rank, self.world, C.byref(self.handle)), "smy_ep_comm_create")

    def close(self):
        if self.handle:
            _lib.load().smy_ep_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class MoELayer:
    """samoyeds_moe_layer with a persistent workspace (graph-capturable).

    comm (EPComm): expert parallelism through the C library's NCCL transport --
    `experts` are then this rank's num_experts / world experts."""

    def __init__(self, cfg: MoEConfig, experts, shared=(), max_tokens: int = 4096, device=None,
                 comm: Optional["EPComm"] = None):
        self.cfg = cfg
        self.comm = comm
        self.experts = experts = prepare_experts(cfg, experts)
        self.shared = shared = prepare_experts(cfg, shared) if shared else shared
        self._arr = _weight_array(experts)
        self._sarr = _weight_array(shared) if shared else None
        self._cfg = cfg.kernel_config().c()
        lib = _lib.load()
        b = C.c_size_t()
        if comm is not None:
            check(lib.smy_moe_ep_workspace_bytes(C.byref(self._cfg), max_tokens, comm.world, C.byref(b)),
                  "smy_moe_ep_workspace_bytes")
        else:
            check(lib.smy_moe_workspace_bytes(C.byref(self._cfg), max_tokens, C.byref(b)),
                  "smy_moe_workspace_bytes")
        self.max_tokens = max_tokens
        self.workspace = torch.empty(b.value, dtype=torch.uint8, device=device or torch.device("cuda"))

    def __call__(self, x: torch.Tensor, logits: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None):
        lib = _lib.load()
        T = x.shape[0]
        if T > self.max_tokens:
            raise ValueError("T exceeds the workspace's max_tokens")
        if out is None:
            out = torch.empty(T, self.cfg.hidden, dtype=torch.bfloat16 if self.cfg.out_dtype == "bf16" else torch.float32,
                              device=x.device)
        xb = x.view(torch.int16) if x.dtype == torch.bfloat16 else x
        check(lib.samoyeds_moe_layer(C.byref(self._cfg), self._arr, self._sarr, _ptr(xb), _ptr(logits), T,
                                     _ptr(out), _ptr(self.workspace), self.workspace.numel(),
                                     self.comm.handle if self.comm is not None else None,
                                     _stream(stream)), "samoyeds_moe_layer")
        return out

    VARIANTS = {"product": 0, "permute": 1, "dense_inter": 2}

    @contextlib.contextmanager
    def variant(self, name: str, T: int):
        """Ablation only (smy_moe_set_variant): inside the block,
        this thread's single-GPU layer calls over <= T tokens run the named
        variant ("permute": materialised input permutation; "dense_inter": token-
        position intermediate layout) with scratch allocated here."""
        lib = _lib.load()
        v = self.VARIANTS[name]
        b = C.c_size_t()
        check(lib.smy_moe_variant_scratch_bytes(C.byref(self._cfg), T, v, C.byref(b)), "smy_moe_variant_scratch_bytes")
        scratch = torch.empty(max(b.value, 1), dtype=torch.uint8, device=self.workspace.device)
        check(lib.smy_moe_set_variant(v, _ptr(scratch), b.value), "smy_moe_set_variant")
        try:
            yield self
        finally:
            check(lib.smy_moe_set_variant(0, None, 0), "smy_moe_set_variant")
            del scratch

    def kernel_names(self, T: int):
        """smy_moe_kernel_names: (gate/up, down) SSMM kernel names of a call over T tokens."""
        lib = _lib.load()
        gu, dn = C.create_string_buffer(96), C.create_string_buffer(96)
        check(lib.smy_moe_kernel_names(C.byref(self._cfg), T, gu, dn, 96), "smy_moe_kernel_names")
        return gu.value.decode(), dn.value.decode()

    def view(self, T: int):
        """smy_moe_workspace_view: the routing result and the compact bf16 gate/up
        intermediate the last single-GPU call over T tokens left in the
        workspace, as views of it: dict counts / offsets / sel / gw / inter
        ([inter_rows x ffn], int16 bf16 bits)."""
        if self.comm is not None:
            raise ValueError("view() describes the single-GPU layer's workspace")
        lib = _lib.load()
        v = _lib.smy_moe_view()
        check(lib.smy_moe_workspace_view(C.byref(self._cfg), T, _ptr(self.workspace), self.workspace.numel(),
                                         C.byref(v)), "smy_moe_workspace_view")
        base = self.workspace.data_ptr()

        def at(ptr, n, dtype, esize):
            off = ptr - base
            return self.workspace[off:off + n * esize].view(dtype)

        g, rows = v.groups, v.inter_rows
        return {"counts": at(v.counts, g, torch.int32, 4), "offsets": at(v.offsets, g + 1, torch.int32, 4),
                "sel": at(v.sel, rows, torch.int32, 4), "gw": at(v.gw, rows, torch.float32, 4),
                "inter": at(v.inter, rows * self.cfg.ffn, torch.int16, 2).view(rows, self.cfg.ffn)}


def synth_fill(out: torch.Tensor, seed: int, dist: int, scale: float, lo: int = -2, hi: int = 2,
               idx0: int = 0, stream=None) -> torch.Tensor:
    """Counter-based generator twin of synth/ (input preparation)."""
    lib = _lib.load()
    bf = out.dtype in (torch.bfloat16, torch.int16)
    check(lib.smy_synth_fill(seed, dist, scale, lo, hi, idx0, out.numel(), _ptr(out), int(bf), _stream(stream)),
          "smy_synth_fill")
    return out


# ------------------------------------------------------------ expert parallelism

def ep_plan(ids: torch.Tensor, w: torch.Tensor, num_experts: int, world: int, stream=None):
    """samoyeds_ep_plan: per-destination send order + tags (see include/samoyeds.h)."""
    lib = _lib.load()
    T, k = ids.shape
    dev = ids.device
    b = C.c_size_t()
    check(lib.smy_ep_plan_workspace_bytes(T, k, world, C.byref(b)), "smy_ep_plan_workspace_bytes")
    ws = torch.empty(b.value, dtype=torch.uint8, device=dev)
    counts = torch.empty(world, dtype=torch.int32, device=dev)
    offsets = torch.empty(world + 1, dtype=torch.int32, device=dev)
    n = max(T * k, 1)
    sel = torch.empty(n, dtype=torch.int32, device=dev)
    tag_ids = torch.empty(n, k, dtype=torch.int32, device=dev)
    tag_w = torch.empty(n, k, dtype=torch.float32, device=dev)
    check(lib.samoyeds_ep_plan(_ptr(ids), _ptr(w), T, k, num_experts, world, _ptr(counts), _ptr(offsets), _ptr(sel),
                               _ptr(tag_ids), _ptr(tag_w), _ptr(ws), ws.numel(), _stream(stream)), "samoyeds_ep_plan")
    return counts, offsets, sel, tag_ids, tag_w


def ep_pack(x: torch.Tensor, offsets: torch.Tensor, sel: torch.Tensor, rows: int, stream=None) -> torch.Tensor:
    lib = _lib.load()
    xb = x.view(torch.int16) if x.dtype == torch.bfloat16 else x
    out = torch.empty(max(rows, 0), xb.shape[1], dtype=torch.int16, device=x.device)
    check(lib.samoyeds_ep_pack(_ptr(xb), xb.stride(0), xb.shape[1], _ptr(offsets), offsets.numel() - 1, _ptr(sel),
                               rows, _ptr(out) if rows > 0 else None, _stream(stream)), "samoyeds_ep_pack")
    return out


def ep_row_ids(sel: torch.Tensor, offsets: torch.Tensor, rank: int, rows: int, stream=None) -> torch.Tensor:
    """samoyeds_ep_row_ids: (rank << 24) | token id of every send row."""
    lib = _lib.load()
    out = torch.empty(max(rows, 1), dtype=torch.int32, device=sel.device)
    check(lib.samoyeds_ep_row_ids(_ptr(sel), _ptr(offsets), offsets.numel() - 1, rank, rows,
                                  _ptr(out), _stream(stream)), "samoyeds_ep_row_ids")
    return out


def ep_combine(back: torch.Tensor, offsets: torch.Tensor, sel: torch.Tensor, out: torch.Tensor, stream=None):
    lib = _lib.load()
    rows = back.shape[0]
    check(lib.samoyeds_ep_combine(_ptr(back) if rows else None, out.shape[1], _ptr(offsets), offsets.numel() - 1,
                                  _ptr(sel), rows, _ptr(out), _stream(stream)), "samoyeds_ep_combine")
    return out


class MoEExperts:
    """samoyeds_moe_experts: the layer body for rows whose routing is given
    (keys = expert ids, -1 = none; vals = gate weights)."""

    def __init__(self, cfg: MoEConfig, experts, max_rows: int, device=None):
        self.cfg = cfg
        self.experts = experts = prepare_experts(cfg, experts)
        self._arr = _weight_array(experts)
        self._cfg = cfg.kernel_config().c()
        lib = _lib.load()
        b = C.c_size_t()
        check(lib.smy_moe_workspace_bytes(C.byref(self._cfg), max_rows, C.byref(b)), "smy_moe_workspace_bytes")
        self.max_rows = max_rows
        self.workspace = torch.empty(b.value, dtype=torch.uint8, device=device or torch.device("cuda"))

    def __call__(self, x: torch.Tensor, keys: torch.Tensor, vals: torch.Tensor, out: Optional[torch.Tensor] = None,
                 stream=None):
        lib = _lib.load()
        R = x.shape[0]
        if R > self.max_rows:
            raise ValueError("rows exceed the workspace's max_rows")
        if out is None:
            out = torch.empty(R, self.cfg.hidden, dtype=torch.float32, device=x.device)
        xb = x.view(torch.int16) if x.dtype == torch.bfloat16 else x
        check(lib.samoyeds_moe_experts(C.byref(self._cfg), self._arr, _ptr(xb) if R else None, R,
                                       _ptr(keys) if R else None, _ptr(vals) if R else None, _ptr(out),
                                       _ptr(self.workspace), self.workspace.numel(), _stream(stream)),
              "samoyeds_moe_experts")
        return out

    def peer(self, world: int, x_ptrs, ldx: int, out_ptrs, ldo: int, row_map: torch.Tensor, keys: torch.Tensor,
             vals: torch.Tensor, stream=None) -> None:
        """samoyeds_moe_experts_peer: received rows read from / reduced into the
        ranks' peer-mapped buffers (x_ptrs / out_ptrs: device pointers valid on
        this device, one per rank)."""
        lib = _lib.load()
        R = row_map.shape[0]
        if R > self.max_rows:
            raise ValueError("rows exceed the workspace's max_rows")
        xp = (C.c_void_p * world)(*[C.c_void_p(p) for p in x_ptrs])
        op = (C.c_void_p * world)(*[C.c_void_p(p) for p in out_ptrs])
        check(lib.samoyeds_moe_experts_peer(C.byref(self._cfg), self._arr, world, xp, ldx, op, ldo, R,
                                            _ptr(row_map) if R else None, _ptr(keys) if R else None,
                                            _ptr(vals) if R else None, _ptr(self.workspace),
                                            self.workspace.numel(), _stream(stream)), "samoyeds_moe_experts_peer")
