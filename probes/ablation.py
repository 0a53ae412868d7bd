"""B200 breakdown ablation of one Mixtral-8x7B expert FFN (the
shape of the paper's Fig. 17 / Fig. 11b breakdown):

  dense            cuBLAS bf16: x[sel] gathered (index_select), gate / up GEMMs,
                   SiLU*up, down GEMM, weighted index_add into the output
  + 2:4 weights    our SSMM, weight-only sparsity (format (2,2,32): N = M), rows
                   read through SEL, SiLU*up as a separate pass, scatter-add epilogue
  + vector-wise    the Samoyeds (1,2,32) format, same launches
  + fused SiLU*up  one SSMM over the interleaved gate/up weight with the SiLU*up
                   epilogue (the layer's path)

n routed tokens of a 4096-token batch (n = 1024: top-2 of 8 experts); ms = median
of 9 runs, L2 flushed before each.  Separate passes (gather, SiLU*up, index_add)
run as torch ops in this probe only -- the product path is all library kernels.

    python probes/ablation.py > profiles/r1_ablation.md
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402

d, f, T = 4096, 14336, 4096


def timed(fn, flush, reps=9):
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
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    x = torch.empty(T, d, dtype=torch.int16, device=dev)
    P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    xb = x.view(torch.bfloat16)
    dense = []
    for i, (r, c) in enumerate(((f, d), (f, d), (d, f))):
        w = torch.empty(r, c, dtype=torch.int16, device=dev)
        P.synth_fill(w, synth.weight_seed(0, i), synth.DIST_UNIFORM, float(synth.uniform_scale(np.sqrt(3.0 / c))))
        dense.append(w)
    rows = []
    for n in (256, 1024, 4096):
        sel = torch.from_numpy(synth.selection(5, T, n)).to(dev)
        sel64 = sel.long()
        g = torch.rand(n, device=dev, dtype=torch.float32)
        out = torch.zeros(T, d, dtype=torch.float32, device=dev)
        wg, wu, wd = (w.view(torch.bfloat16) for w in dense)

        def run_dense():
            xs = torch.index_select(xb, 0, sel64)
            a = torch.nn.functional.silu(xs @ wg.t()) * (xs @ wu.t())
            out.index_add_(0, sel64, (a @ wd.t()).float() * g[:, None])

        res = {"n": n, "dense (cuBLAS)": timed(run_dense, flush)}
        for name, fmt in (("+ 2:4 weights (2,2,32)", P.Format(2, 2, 32)), ("+ vector-wise (1,2,32)", P.Format(1, 2, 32))):
            sg, su, sd = (P.compress(w, fmt)[0] for w in dense)

            def run_sparse():
                h = P.ssmm(sg, x, sel, out_dtype=torch.bfloat16)
                u = P.ssmm(su, x, sel, out_dtype=torch.bfloat16)
                a = (torch.nn.functional.silu(h.float()) * u.float()).to(torch.bfloat16)
                P.ssmm(sd, a.view(torch.int16), torch.arange(n, device=dev, dtype=torch.int32), epi="scatter_add",
                       scale=g, out=out)   # rows 0..n-1 of `out` (the destination map is the probe's concern)
            res[name] = timed(run_sparse, flush)
            if fmt.n == 1:
                gu = P.interleave_gate_up(sg, su)
                idx = torch.arange(n, device=dev, dtype=torch.int32)

                def run_fused():
                    a = P.ssmm(gu, x, sel, epi="silu_mul_interleaved")
                    P.ssmm(sd, a.view(torch.int16), idx, epi="scatter_add", scale=g, out=out)
                res["+ fused SiLU*up (interleaved)"] = timed(run_fused, flush)
        rows.append(res)
        print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}, file=sys.stderr, flush=True)
    cols = [c for c in rows[0] if c != "n"]
    print("# Breakdown ablation, one Mixtral-8x7B expert FFN on B200 (probes/ablation.py)\n")
    print("ms per expert FFN (gate, up, SiLU*up, down + weighted accumulation), n routed tokens of 4096; "
          "speed-up over dense cuBLAS in brackets.\n")
    print("| n | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows:
        base = r["dense (cuBLAS)"]
        print(f"| {r['n']} | " + " | ".join(f"{r[c]:.3f} ({base / r[c]:.2f}x)" for c in cols) + " |")


if __name__ == "__main__":
    main()
