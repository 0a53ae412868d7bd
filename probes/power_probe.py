"""SM clock and board power while the layer (and its ablation variants) run back to
back for a few seconds each: is the gate/up gap between the SEL gather and the
materialised permutation a power-cap (clock) effect?  nvidia-smi sampled every
50 ms by bench.ClockSampler; the layer call is timed with CUDA events meanwhile.

    python probes/power_probe.py mixtral 4096 [seconds]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    secs = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
    d, f, E, k, gating = bench.MODELS[model]
    dev = torch.device("cuda")
    layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, gating, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                       max_tokens=T, device=dev)
    x = torch.empty(T, d, dtype=torch.int16, device=dev)
    P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    lg = torch.empty(T, E, dtype=torch.float32, device=dev)
    P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    out = torch.empty(T, d, dtype=torch.float32, device=dev)

    def run(name):
        for _ in range(5):
            layer(x, lg, out)
        torch.cuda.synchronize()
        smp = bench.ClockSampler(0)
        smp.start()
        t0 = time.time()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        a.record()
        while time.time() - t0 < secs:
            for _ in range(10):
                layer(x, lg, out)
            n += 10
            torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        t1 = time.time()
        smp.stop(t0, t1)
        rows = [ln.split(",") for _, ln in smp.lines if ln]
        mhz = [float(r[0]) for r in rows if len(r) > 2 and r[0].strip().replace(".", "").isdigit()]
        pw = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        print("%-12s %.4f ms/call  SM clock median %s MHz (min %s)  power median %s W  samples %d" % (
            name, a.elapsed_time(b) / n, np.median(mhz) if mhz else None, min(mhz) if mhz else None,
            np.median(pw) if pw else None, len(mhz)), flush=True)

    run("product")
    for v in ("permute", "dense_inter"):
        with layer.variant(v, T):
            run(v)
    run("product")


if __name__ == "__main__":
    main()
