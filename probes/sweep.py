"""SSMM shape / sparsity sweep on the B200 (BASELINE.json config 5; SURVEY.md §8(d)
config 5 and §8(f)-2's breakdown): our kernels against dense bf16 cuBLAS.

For each (M rows, K, n routed tokens of a pool of 16384 token rows), one GEMM
C[n x M] = x[sel] W^T, bf16 in, fp32 accumulate:
  cublas+gather  torch.index_select(x, sel) then torch.matmul (dense bf16, cuBLAS)
  cublas         torch.matmul on pre-gathered rows (the gather excluded)
  ssmm 2:4       our SSMM on the weight pruned to plain 2:4 -- format (2,2,32), N = M:
                 weight-only sparsity, rows read through SEL (no vector-wise remap)
  ssmm (1,2,32)  our SSMM on the Samoyeds format (vector-wise + 2:4, 75 % sparse),
                 rows read through SEL  -- the paper's dual-side sparse kernel
  ssmm (1,2,16)  same at V = 16, run as its plain-2:4 transcode (the layer's path)
  cusparselt     the vendor weight-only 2:4 kernel (cuSPARSELt through torch's
                 to_sparse_semi_structured) on pre-gathered rows -- TIMING ONLY: torch's
                 binding returns wrong values on this box (probes/cslt_dbg.py)
Every kernel writes fp32 [n x M].  Timing: CUDA events around the op only,
median of R iterations, L2 flushed (a 512 MB memset) before each.
Useful TFLOP/s follow SURVEY §8(d): 2 * (M * N/M_fmt) * K * n for ours (the
dense-equivalent work of the retained sub-rows -- the convention of the 2:4
"sparse peak"), 2 * M * K * n for dense; `eff_tflops` = 2 M K n / t for all.

    python probes/sweep.py [--quick] > profiles/r1_sweep.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402

POOL = 16384


def timed(fn, flush, reps):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    dev = torch.device("cuda")
    Ms = [4096, 14336] if args.quick else [1024, 4096, 14336]
    Ks = [4096, 14336] if args.quick else [1024, 4096, 14336]
    ns = [256, 4096, 16384] if args.quick else [256, 2048, 8192, 16384]
    fmts = {"ssmm_2:4 (2,2,32)": P.Format(2, 2, 32), "ssmm (1,2,32)": P.Format(1, 2, 32),
            "ssmm (1,2,16)": P.Format(1, 2, 16)}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rows = []
    for K in Ks:
        x = torch.empty(POOL, K, dtype=torch.int16, device=dev)
        P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
        xb = x.view(torch.bfloat16)
        for M in Ms:
            wt = torch.empty(M, K, dtype=torch.int16, device=dev)
            P.synth_fill(wt, synth.weight_seed(0, 0), synth.DIST_UNIFORM,
                         float(synth.uniform_scale(np.sqrt(3.0 / K))))
            wd = wt.view(torch.bfloat16)
            sws = {name: P.compress(wt, fmt)[0] for name, fmt in fmts.items()}
            try:
                from torch.sparse import SparseSemiStructuredTensor, to_sparse_semi_structured
                SparseSemiStructuredTensor._FORCE_CUTLASS = False
                g = wd.float().view(M, K // 4, 4)
                keep = torch.zeros_like(g, dtype=torch.bool).scatter_(-1, g.abs().topk(2, dim=-1).indices, True)
                w24 = to_sparse_semi_structured((g * keep).view(M, K).to(torch.bfloat16))
            except Exception as exc:  # no cuSPARSELt: the column stays empty
                print("cusparselt unavailable:", repr(exc)[:120], file=sys.stderr)
                w24 = None
            # V=16 has no fast kernel of its own: the library's path is its plain-2:4 transcode
            sws["ssmm (1,2,16)"] = P.transcode_24(sws["ssmm (1,2,16)"])
            for sw in sws.values():
                sw.drop_canonical()
            for n in ns:
                sel = torch.from_numpy(synth.selection(5, POOL, n)).to(dev)
                out = torch.empty(n, M, dtype=torch.float32, device=dev)
                xs = torch.index_select(xb, 0, sel.long())
                r = {"M": M, "K": K, "n": n, "routed_fraction": n / POOL, "ms": {}}
                r["ms"]["cublas+gather"] = timed(lambda: torch.matmul(torch.index_select(xb, 0, sel.long()), wd.t(),
                                                                      out=None), flush, args.reps)
                r["ms"]["cublas"] = timed(lambda: torch.matmul(xs, wd.t()), flush, args.reps)
                if w24 is not None:
                    xst = xs.t().contiguous()
                    r["ms"]["cusparselt"] = timed(lambda: torch.mm(w24, xst), flush, args.reps)
                for name, sw in sws.items():
                    r["ms"][name] = timed(lambda: P.ssmm(sw, x, sel, out=out), flush, args.reps)
                dense_flops = 2.0 * M * K * n
                r["eff_tflops"] = {k: dense_flops / (v * 1e-3) / 1e12 for k, v in r["ms"].items()}
                r["useful_tflops"] = {k: (dense_flops * (fmts[k].n / fmts[k].m) if k in fmts else
                                          dense_flops / 2 if k == "cusparselt" else dense_flops)
                                      / (v * 1e-3) / 1e12 for k, v in r["ms"].items()}
                r["speedup_vs_cublas_gather"] = {k: r["ms"]["cublas+gather"] / v for k, v in r["ms"].items()}
                rows.append(r)
                print(json.dumps({"M": M, "K": K, "n": n, **{k: round(v, 4) for k, v in r["ms"].items()}}),
                      file=sys.stderr, flush=True)
            del sws, wt, w24
        del x
    print(json.dumps({"_note": __doc__.strip().splitlines()[0], "device": torch.cuda.get_device_name(),
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
