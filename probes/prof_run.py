"""SMY_DEBUG=128: per-role cycle counters of the 2-CTA pair kernel on the bench workload."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
lib = P.load()
d, f, E, k, g = bench.MODELS[model]
dev = torch.device("cuda")
layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, g, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                   max_tokens=T, device=dev)
x = torch.empty(T, d, dtype=torch.int16, device=dev)
P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
lg = torch.empty(T, E, dtype=torch.float32, device=dev)
P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
out = torch.empty(T, d, dtype=torch.float32, device=dev)
import contextlib
variant = sys.argv[3] if len(sys.argv) > 3 else None
ctx = layer.variant(variant, T) if variant else contextlib.nullcontext()
ctx.__enter__()
for _ in range(3):
    layer(x, lg, out)
buf = (C.c_ulonglong * (148 * 32))()
lib.smy_debug_prof(buf, 148)
R = 5
for _ in range(R):
    layer(x, lg, out)
lib.smy_debug_prof(buf, 148)
raw = np.array(buf, dtype=np.float64).reshape(2, 148, 16)
A = raw / R / 1e3
for name, a in zip(("gate/up", "down"), A):
    lead = a[0::2]
    t = max(lead[:, 7].mean(), 1e-9)
    print(f"{model} T={T} {name}: kcycles per CTA per layer call; tiles/pair {lead[:, 7].mean() * 1e3:.1f}")
    print("  MMA warp: total %.1f  wait_full %.1f (token ring %.1f)  wait_acc_empty %.1f  issue %.1f"
          % (lead[:, 2].mean(), lead[:, 0].mean(), lead[:, 6].mean(), lead[:, 1].mean(),
             (lead[:, 2] - lead[:, 0] - lead[:, 1]).mean()))
    print("  gather warp: wait_empty %.1f  issue %.1f (leader) / %.1f %.1f (peer)"
          % (lead[:, 10].mean(), lead[:, 11].mean(), a[1::2, 10].mean(), a[1::2, 11].mean()))
    r = raw[0 if name == "gate/up" else 1]
    live = r[:, 14] > 0
    if live.any():
        st, en = r[live, 14], r[live, 15]
        print("  CTA lifetime %.1f us (mean), max %.1f us; last call: CTA starts spread %.1f us, ends spread %.1f us,"
              " span %.1f us" % (a[:, 13].mean(), a[:, 13].max(), (st.max() - st.min()) / 1e3,
                                 (en.max() - en.min()) / 1e3, (en.max() - st.min()) / 1e3))
    print("  epilogue: wait_acc_full %.1f  work %.1f (tmem_ld %.1f)   producer wait_empty %.1f"
          % tuple(a[:, i].mean() for i in (3, 4, 8, 5)))
    if lead[:, 12].mean() > 0:
        ks = {"mixtral": 32, "qwen2": 28, "deepseek": 16}.get(model, 1)
        n = lead[:, 7].mean() * ks
        print("  token slot (leader): issue -> ready seen by the MMA %.0f clk, slot round trip %.0f clk (per stage)"
              % (lead[:, 12].mean() * 1e3 / n, lead[:, 9].mean() * 1e3 / n))
