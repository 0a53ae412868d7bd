"""ctypes binding of libsamoyeds.so (include/samoyeds.h).  Marshalling only.

Loading fails loudly: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# SMY_LIB_PATH: load another build of the same library (A/B experiments in probes/)
LIB_PATH = os.environ.get("SMY_LIB_PATH") or os.path.join(_PKG, "libsamoyeds.so")


class smy_format(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("v", C.c_int32)]


class smy_wdesc(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("fmt", smy_format)]


class smy_wlayout(C.Structure):
    _fields_ = [("values", C.c_size_t), ("codes", C.c_size_t), ("indices", C.c_size_t), ("image", C.c_size_t),
                ("comp_rows", C.c_int32), ("m_tiles", C.c_int32), ("k_stages", C.c_int32),
                ("planes", C.c_int32), ("rep", C.c_int32), ("block", C.c_int32)]


class smy_weight(C.Structure):
    _fields_ = [("d", smy_wdesc), ("values", C.c_void_p), ("codes", C.c_void_p), ("indices", C.c_void_p),
                ("image", C.c_void_p)]


class smy_moe_config(C.Structure):
    _fields_ = [("num_experts", C.c_int32), ("top_k", C.c_int32), ("hidden", C.c_int32), ("ffn", C.c_int32),
                ("num_shared", C.c_int32), ("gating", C.c_int32), ("fmt", smy_format), ("gate_up", C.c_int32),
                ("out_dtype", C.c_int32)]


class smy_moe_view(C.Structure):
    _fields_ = [("counts", C.c_void_p), ("offsets", C.c_void_p), ("sel", C.c_void_p), ("gw", C.c_void_p),
                ("inter", C.c_void_p), ("inter_rows", C.c_int64), ("groups", C.c_int32)]


# name -> (restype, argtypes)
SIGNATURES = {
    "smy_status_str": (C.c_char_p, [C.c_int]),
    "smy_version": (C.c_int, []),
    "smy_last_error": (C.c_char_p, []),
    "smy_weight_layout": (C.c_int, [C.POINTER(smy_wdesc), C.POINTER(smy_wlayout)]),
    "samoyeds_compress": (C.c_int, [C.POINTER(smy_wdesc), C.c_void_p, C.c_int64, C.c_int, C.POINTER(smy_weight),
                                    C.c_void_p, C.c_void_p]),
    "samoyeds_decompress": (C.c_int, [C.POINTER(smy_weight), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "samoyeds_validate_sel": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]),
    "samoyeds_interleave_gate_up": (C.c_int, [C.POINTER(smy_weight), C.POINTER(smy_weight), C.POINTER(smy_weight),
                                              C.c_void_p]),
    "samoyeds_ssmm": (C.c_int, [C.POINTER(smy_weight), C.POINTER(smy_weight), C.c_void_p, C.c_int64, C.c_int64,
                                C.c_void_p, C.c_int32, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                C.c_void_p]),
    "smy_route_workspace_bytes": (C.c_int, [C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]),
    "samoyeds_route": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                 C.c_void_p]),
    "smy_moe_workspace_bytes": (C.c_int, [C.POINTER(smy_moe_config), C.c_int64, C.POINTER(C.c_size_t)]),
    "samoyeds_moe_layer": (C.c_int, [C.POINTER(smy_moe_config), C.POINTER(smy_weight), C.POINTER(smy_weight),
                                     C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t,
                                     C.c_void_p, C.c_void_p]),
    "smy_ep_plan_workspace_bytes": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
    "samoyeds_ep_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                   C.c_void_p]),
    "samoyeds_ep_pack": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_void_p]),
    "samoyeds_moe_experts": (C.c_int, [C.POINTER(smy_moe_config), C.POINTER(smy_weight), C.c_void_p, C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "samoyeds_ep_combine": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p]),
    "samoyeds_ep_row_ids": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                      C.c_void_p]),
    "samoyeds_moe_experts_peer": (C.c_int, [C.POINTER(smy_moe_config), C.POINTER(smy_weight), C.c_int32,
                                            C.POINTER(C.c_void_p), C.c_int64, C.POINTER(C.c_void_p), C.c_int64,
                                            C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                            C.c_void_p]),
    "smy_ep_unique_id": (C.c_int, [C.c_void_p]),
    "smy_ep_comm_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "smy_ep_comm_destroy": (C.c_int, [C.c_void_p]),
    "smy_moe_ep_workspace_bytes": (C.c_int, [C.POINTER(smy_moe_config), C.c_int64, C.c_int32,
                                             C.POINTER(C.c_size_t)]),
    "smy_moe_kernel_names": (C.c_int, [C.POINTER(smy_moe_config), C.c_int64, C.c_char_p, C.c_char_p, C.c_int32]),
    "smy_moe_workspace_view": (C.c_int, [C.POINTER(smy_moe_config), C.c_int64, C.c_void_p, C.c_size_t,
                                         C.POINTER(smy_moe_view)]),
    "smy_moe_set_phase_events": (C.c_int, [C.c_void_p, C.c_int]),
    "smy_moe_variant_scratch_bytes": (C.c_int, [C.POINTER(smy_moe_config), C.c_int64, C.c_int32,
                                               C.POINTER(C.c_size_t)]),
    "smy_moe_set_variant": (C.c_int, [C.c_int32, C.c_void_p, C.c_size_t]),
    "smy_launch_count": (C.c_uint64, []),
    "smy_debug_prof": (C.c_int, [C.c_void_p, C.c_int]),
    "smy_synth_fill": (C.c_int, [C.c_uint64, C.c_int, C.c_float, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                 C.c_void_p, C.c_int, C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2503_10725_b200.build` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class SamoyedsError(RuntimeError):
    def __init__(self, status: int, where: str):
        lib = load()
        msg = lib.smy_status_str(status).decode()
        detail = lib.smy_last_error().decode()
        super().__init__(f"{where}: {msg}" + (f" ({detail})" if detail else ""))
        self.status = status


def check(status: int, where: str) -> None:
    if status != 0:
        raise SamoyedsError(status, where)
