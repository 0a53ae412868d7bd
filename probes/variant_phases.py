"""Per-phase times (route | gate/up | down) of the layer and its ablation variants
(smy_moe_set_variant): how much of the gate/up time is the SEL gather vs the
contiguous-TMA read of a materialised permutation.  SMY_DEBUG bits 1/2 (no gather
/ no weight copies; results garbage) can be set in the environment to bound the
data movement.

    python probes/variant_phases.py mixtral 4096
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    d, f, E, k, gating = bench.MODELS[model]
    dev = torch.device("cuda")
    lib = P.load()
    layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, gating, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                       max_tokens=T, device=dev)
    x = torch.empty(T, d, dtype=torch.int16, device=dev)
    P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    lg = torch.empty(T, E, dtype=torch.float32, device=dev)
    P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
    out = torch.empty(T, d, dtype=torch.float32, device=dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    s = torch.cuda.current_stream()
    for e in evs:
        e.record(s)
    torch.cuda.synchronize()
    h = bench.C_void_p_array(evs)

    def phases(reps=20):
        for _ in range(3):
            layer(x, lg, out)
        r = []
        for _ in range(reps):
            lib.smy_moe_set_phase_events(h, 6)
            layer(x, lg, out)
            lib.smy_moe_set_phase_events(None, 0)
            torch.cuda.synchronize()
            r.append([evs[i].elapsed_time(evs[i + 1]) for i in range(5)])
        m = np.median(np.array(r), axis=0)
        return {"route": round(m[0], 4), "gate_up": round(m[2], 4), "down(+unpermute)": round(m[3], 4)}
    print(model, T, "SMY_DEBUG=%s" % os.environ.get("SMY_DEBUG", "0"))
    print("  product      ", phases())
    for v in ("permute", "dense_inter"):
        with layer.variant(v, T):
            print("  %-13s" % v, phases())


if __name__ == "__main__":
    main()
