"""Run a fixed set of GPU parity tests by node id (for compute-sanitizer; probes/sanitize.sh)."""
import sys

import pytest

T = "tests/test_gpu_parity.py::"
SETS = {
    "1": [T + "test_moe_layer_parity[SparseFormat(n=1, m=2, v=32)-E8-T100-auto-auto-sh0]",
          T + "test_moe_layer_parity[SparseFormat(n=1, m=2, v=32)-E16-T257-auto-auto-sh2]"],
    "2": [T + "test_moe_layer_prefill_pair_kernels[E4-d512-f512-T512-auto-sh0]",
          T + "test_moe_layer_prefill_pair_kernels[E4-d256-f640-T400-auto-sh0]"],
    "3": [T + "test_ssmm_random_tolerance[shape1-SparseFormat(n=1, m=2, v=32)]",
          T + "test_ssmm_random_tolerance[shape3-SparseFormat(n=1, m=2, v=32)]",
          T + "test_ssmm_random_tolerance[shape2-SparseFormat(n=2, m=2, v=32)]"],
    # the (N, 2N, 32) row expansion (XP) and the pair kernel's extra epilogue warps (down)
    "4": [T + "test_ssmm_expanded_integer_exact[scatter_add-SparseFormat(n=4, m=8, v=32)]",
          T + "test_ssmm_silu_mul_interleaved_expanded[shape1-SparseFormat(n=8, m=16, v=32)]",
          T + "test_moe_layer_parity[SparseFormat(n=4, m=8, v=32)-E8-T7-auto-off-sh0]",
          T + "test_moe_layer_prefill_pair_kernels[E4-d512-f512-T512-auto-sh0]"],
}
sys.exit(pytest.main(["-x", "-q", "-p", "no:cacheprovider"] + SETS[sys.argv[1]]))
