"""B200-native (sm_100a) implementation of the Samoyeds hot path (arXiv 2503.10725):
dual-side sparse SSMM of MoE expert FFNs behind the C ABI in include/samoyeds.h.

The compute path is libsamoyeds.so (csrc/); this package is the thin Python
binding over it.  There is no CPU fallback: importing the API without the
built library raises.
"""
from .api import (EPComm, MoEConfig, MoEExperts, MoELayer, Format, SparseWeight, compress, decompress, transcode_24, ep_combine, ep_pack,  # noqa: F401
                  ep_plan, ep_row_ids, interleave_gate_up, prepare_experts, route, ssmm, synth_fill, validate_sel,
                  weight_layout)
from . import ep  # noqa: F401
from ._lib import LIB_PATH, SamoyedsError, load  # noqa: F401
