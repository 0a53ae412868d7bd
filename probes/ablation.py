"""B200 breakdown of the Samoyeds MoE layer: the paper's step-by-step
ablation (Fig. 17) and its compressed-output-layout figure (Fig. 11b,
P:374-376), on whole MoE layers of the BASELINE models at T tokens.

  vanilla      dense bf16 cuBLAS (torch.mm per expert), the input PERMUTED into an
               expert-major copy (index_select), SiLU*up, down, weighted index_add
               un-permute -- one CUDA graph (routing precomputed, static shapes)
  +W           weight sparsity: the library layer in SMY_VARIANT_PERMUTE -- the same
               permute / un-permute passes around our (1,2,32) SSMMs (gate/up reads the
               permuted copy as contiguous rows through 2D TMA)
  +WI          + input sparsity: SSMM gathering x through SEL, weighted scatter-add into
               the output (no permutation passes) -- but the gate/up intermediate in a
               token-position layout [E x T x f], zero-filled every call
               (SMY_VARIANT_DENSE_INTER: the layout P:374 replaces)
  +WIT         + the compressed output layout: the product layer (compact bf16
               intermediate aligned with SEL)

The data-stationary remap (S) is inherent in every sparse column here
(lane-masked accumulator slots), so it has no column of its own.
ms = median of CUDA-event-timed replays (weights >> L2, streamed every call);
routing time excluded from vanilla, included in the library columns (it is a few
us).  Layout figure: dense_inter vs compact at the model's routed density k/E.

    python probes/ablation.py > profiles/r2_ablation.md
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def vanilla(model, T, x, lg, dev):
    d, f, E, k, gating = bench.MODELS[model]
    ws = []
    for e in range(E):
        trip = []
        for i in range(3):
            r, c = (f, d) if i < 2 else (d, f)
            w = torch.empty(r, c, dtype=torch.int16, device=dev)
            P.synth_fill(w, synth.weight_seed(e, i), synth.DIST_UNIFORM, float(synth.uniform_scale(np.sqrt(3.0 / c))))
            trip.append(w.view(torch.bfloat16))
        ws.append(trip)
    ids, gw = P.route(lg, k, gating)[:2]
    flat = ids.flatten().long()
    order = torch.argsort(flat, stable=True)                 # expert-major permutation
    tok = (order // k).to(dev)
    g = gw.flatten()[order].float()
    counts = torch.bincount(flat, minlength=E).cpu().tolist()
    xb = x.view(torch.bfloat16)
    out = torch.zeros(T, d, dtype=torch.float32, device=dev)
    xp = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)
    y = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)

    def step():
        out.zero_()
        torch.index_select(xb, 0, tok, out=xp)
        o = 0
        for e, n in enumerate(counts):
            if n:
                xs = xp[o:o + n]
                a = torch.nn.functional.silu(xs @ ws[e][0].t()) * (xs @ ws[e][1].t())
                torch.mm(a, ws[e][2].t(), out=y[o:o + n])
            o += n
        out.index_add_(0, tok, y.float() * g[:, None])

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    t = timed(graph.replay)
    del ws, graph
    torch.cuda.empty_cache()
    return t


def main():
    dev = torch.device("cuda")
    rows = []
    cases = [("mixtral", 4096), ("qwen2", 4096), ("deepseek", 4096), ("mixtral", 1024)]
    for model, T in cases:
        d, f, E, k, gating = bench.MODELS[model]
        x = torch.empty(T, d, dtype=torch.int16, device=dev)
        P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
        lg = torch.empty(T, E, dtype=torch.float32, device=dev)
        P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
        res = {"model": model, "T": T, "density": k / E}
        res["vanilla"] = vanilla(model, T, x, lg, dev)
        layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, gating, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                           max_tokens=T, device=dev)
        out = torch.empty(T, d, dtype=torch.float32, device=dev)
        ref = layer(x, lg, out).clone()
        for name, v in (("+W", "permute"), ("+WI", "dense_inter")):
            with layer.variant(v, T):
                res[name] = timed(lambda: layer(x, lg, out))
                err = float((out - ref).norm() / ref.norm())
                assert err < 1e-3, (model, v, err)
        res["+WIT"] = timed(lambda: layer(x, lg, out))
        rows.append(res)
        print(res, file=sys.stderr, flush=True)
        del layer
        torch.cuda.empty_cache()
    cols = ["vanilla", "+W", "+WI", "+WIT"]
    print("# Breakdown of the MoE layer on B200 (probes/ablation.py; paper Fig. 17 / Fig. 11b)\n")
    print("ms per layer call (gate/up, SiLU*up, down, weighted accumulation over all experts), "
          "speed-up over vanilla in brackets; the last column is the compact-vs-token-position "
          "intermediate layout speed-up (Fig. 11b analogue) at the model's routed density k/E.\n")
    print("| model | T | k/E | " + " | ".join(cols) + " | +WI -> +WIT (layout) | +W -> +WI (input sparsity) |")
    print("|---|---|---|" + "---|" * (len(cols) + 2))
    for r in rows:
        base = r["vanilla"]
        print(f"| {r['model']} | {r['T']} | {r['density']:.3f} | " +
              " | ".join(f"{r[c]:.3f} ({base / r[c]:.2f}x)" for c in cols) +
              f" | {r['+WI'] / r['+WIT']:.2f}x | {r['+W'] / r['+WI']:.2f}x |")


if __name__ == "__main__":
    main()
