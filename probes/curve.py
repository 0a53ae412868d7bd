"""Throughput-vs-tokens curve of the MoE layer (BASELINE config 2 "batch 1-4096", the
paper's throughput-vs-batch analogue; config 4's Qwen2 token set) with
the roofline fraction of each point.

Every call is timed on its own with CUDA events (one replay of a captured graph
of that single layer call) after L2 is evicted by writing a 256 MB buffer, so
decode points stream their experts' weights from HBM every time (no L2 reuse
between iterations).  Per point: ms, tokens/s, gate/up and down SSMM times (the
layer's phase events, recorded in a second, separate timing), and the fraction of
the bound that applies to each SSMM: HBM (algorithmic bytes / time / measured
HBM GB/s) below the ridge, the 2:4-sparse tensor peak (2 x measured dense bf16)
above it -- the same byte / flop formulas as bench.py.

    python probes/curve.py mixtral 1,2,4,...  > profiles/r2_curve_mixtral.json
    SMY_FORMAT=4,8,32 SMY_TRANSCODE=off python probes/curve.py mixtral ...   (other formats / native images)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402


def main():
    model = sys.argv[1]
    Ts = [int(t) for t in sys.argv[2].split(",")]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    d, f, E, k, gating = bench.MODELS[model]
    if os.environ.get("SMY_FORMAT"):
        bench.set_format(os.environ["SMY_FORMAT"])  # FMT and the per-element byte count
    tc = os.environ.get("SMY_TRANSCODE", "auto")
    dev = torch.device("cuda")
    lib = P.load()
    Tmax = max(Ts)
    layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, gating, P.Format(*bench.FMT), transcode=tc),
                       bench.build_layer(P, model, dev, transcode=tc), max_tokens=Tmax, device=dev)
    x = torch.empty(Tmax, d, dtype=torch.int16, device=dev)
    P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    lg = torch.empty(Tmax, E, dtype=torch.float32, device=dev)
    P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    out = torch.empty(Tmax, d, dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm, burst, _, src = bench.peaks()
    sparse_peak = 2.0 * burst
    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for e in evs:
        e.record(stream)
    torch.cuda.synchronize()
    handles = bench.C_void_p_array(evs)
    res = []
    for T in Ts:
        xs, ls, os_ = x[:T], lg[:T], out[:T]
        for _ in range(3):
            layer(xs, ls, os_)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer(xs, ls, os_)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot, ph = [], []
        for i in range(reps):
            flush.fill_(i & 0xFF)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            tot.append(a.elapsed_time(b))
        for i in range(reps):   # phase split: eager calls recording the layer's events
            flush.fill_(i & 0xFF)
            lib.smy_moe_set_phase_events(handles, 6)
            layer(xs, ls, os_)
            lib.smy_moe_set_phase_events(None, 0)
            torch.cuda.synchronize()
            ph.append([evs[j].elapsed_time(evs[j + 1]) for j in range(5)])
        ms = float(np.median(tot))
        phm = np.median(np.array(ph), axis=0)
        ids = P.route(ls, k, gating)[0].flatten().long()
        cnt = torch.bincount(ids, minlength=E)
        act = int((cnt > 0).sum())
        Tk = T * k
        fl_gu = 2 * 2 * (f // 2) * d * Tk
        by_gu = 2 * act * f * d * bench.BYTES_PER_ELEM + Tk * d * 2 + Tk * 4 + Tk * f * 2
        fl_dn = fl_gu / 2
        by_dn = act * f * d * bench.BYTES_PER_ELEM + Tk * f * 2 + Tk * 8 + Tk * d * 4
        ridge = sparse_peak * 1e12 / (hbm * 1e9)

        def frac(fl, by, t_ms):
            t = t_ms * 1e-3
            if fl / by >= ridge:
                return {"bound": "tensor", "frac": fl / t / 1e12 / sparse_peak, "tflops": fl / t / 1e12}
            return {"bound": "hbm", "frac": by / t / 1e9 / hbm, "gbs": by / t / 1e9}
        r = {"model": model, "T": T, "ms": ms, "tokens_per_s": T / (ms * 1e-3), "active_experts": act,
             "route_ms": float(phm[0]), "gate_up_ms": float(phm[2]), "down_ms": float(phm[3]),
             "gate_up": frac(fl_gu, by_gu, phm[2]), "down": frac(fl_dn, by_dn, phm[3]),
             "layer_hbm_frac": (by_gu + by_dn) / (ms * 1e-3) / 1e9 / hbm,
             "layer_sparse_frac": (fl_gu + fl_dn) / (ms * 1e-3) / 1e12 / sparse_peak}
        res.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
        del g
    json.dump({"model": model, "peaks": {"hbm_gbs": hbm, "sparse_tflops": sparse_peak, "source": src},
               "l2": "256 MB written before every timed call (L2 evicted)", "points": res}, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
