"""cuSPARSELt 2:4 bf16 throughput on this B200: the
vendor weight-only 2:4 baseline (the paper's cuSPARSELt comparison) and
the ground truth for the "2:4 sparse peak = 2 x dense" denominator.

Uses torch's cuSPARSELt binding (torch._cslt_compress / torch._cslt_sparse_mm,
cuSPARSELt 0.7.1 in this image): C[m x n] = W_24[m x k] @ X^T[k x n], bf16 in,
bf16 out, fp32 accumulation, best algorithm from torch's own search
(_cslt_sparse_mm_search).  Same shapes through torch.matmul (dense cuBLAS).

    python probes/cslt_bench.py [--out gpurun_out/cslt.json]
"""
from __future__ import annotations

import argparse
import json

import torch


def timeit(fn, iters=50, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def prune24(w):
    """keep the 2 largest |w| of every 4 consecutive along K"""
    m, k = w.shape
    g = w.view(m, k // 4, 4)
    idx = g.abs().topk(2, dim=-1).indices
    mask = torch.zeros_like(g, dtype=torch.bool).scatter_(-1, idx, True)
    return (g * mask).view(m, k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    torch.manual_seed(0)
    dev = torch.device("cuda")
    rows = []
    shapes = [(8192, 8192, 8192), (16384, 16384, 8192), (14336, 4096, 1024), (14336, 4096, 4096),
              (14336, 4096, 8192), (14336, 4096, 16384), (4096, 14336, 8192), (28672, 4096, 8192),
              (2816, 2048, 4096), (2048, 1408, 4096), (5120, 3584, 4096), (3584, 2560, 4096),
              (14336, 4096, 256), (14336, 4096, 64)]
    for m, k, n in shapes:
        w = prune24(torch.randn(m, k, device=dev, dtype=torch.bfloat16) / k ** 0.5)
        x = torch.randn(n, k, device=dev, dtype=torch.bfloat16)
        xt = x.t().contiguous()
        try:
            # torch's public semi-structured API on the cuSPARSELt backend (handles the
            # operand layouts); C = W_24 @ X^T
            from torch.sparse import SparseSemiStructuredTensor, to_sparse_semi_structured
            SparseSemiStructuredTensor._FORCE_CUTLASS = False
            ws = to_sparse_semi_structured(w)
            ref = w.float() @ xt.float()
            got = torch.mm(ws, xt).float()
            err = float((got - ref).norm() / ref.norm())
            layout = type(ws).__name__
            t_sp = timeit(lambda: torch.mm(ws, xt))
        except Exception as exc:  # report, keep going
            rows.append({"m": m, "k": k, "n": n, "error": repr(exc)[:200]})
            print(rows[-1], flush=True)
            continue
        t_d = timeit(lambda: w @ xt)
        fl = 2.0 * m * k * n
        r = {"m": m, "k": k, "n": n, "cslt_ms": t_sp, "dense_ms": t_d,
             "cslt_tflops_dense_equiv": fl / t_sp / 1e9, "dense_tflops": fl / t_d / 1e9,
             "cslt_speedup": t_d / t_sp, "cslt_rel_err": err, "b_layout": layout}
        rows.append(r)
        print(json.dumps(r), flush=True)
    if args.out:
        json.dump({"torch": torch.__version__, "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
