"""SMY_DEBUG=128 per-role cycle counters of the single-CTA SSMM kernel (all CTAs),
e.g. the (N, 2N, 32) row-expansion kernels: python probes/xp_prof.py mixtral 64 4,8,32 off"""
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
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
bench.FMT = tuple(int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "4,8,32").split(","))
tc = sys.argv[4] if len(sys.argv) > 4 else "off"
lib = P.load()
d, f, E, k, g = bench.MODELS[model]
dev = torch.device("cuda")
cfg = P.MoEConfig(E, k, d, f, 0, g, P.Format(*bench.FMT), "auto", tc)
layer = P.MoELayer(cfg, bench.build_layer(P, model, dev, transcode=tc), max_tokens=T, device=dev)
print("kernels:", layer.kernel_names(T) if hasattr(layer, "kernel_names") else "")
x = torch.empty(T, d, dtype=torch.int16, device=dev)
P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
lg = torch.empty(T, E, dtype=torch.float32, device=dev)
P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
out = torch.empty(T, d, dtype=torch.float32, device=dev)
for _ in range(3):
    layer(x, lg, out)
buf = (C.c_ulonglong * (148 * 32))()
lib.smy_debug_prof(buf, 148)
R = 5
for _ in range(R):
    layer(x, lg, out)
torch.cuda.synchronize()
lib.smy_debug_prof(buf, 148)
a = np.array(buf, dtype=np.float64).reshape(2, 148, 16) / R / 1e3
for name, r in zip(("gate/up", "down"), a):
    m = r.mean(axis=0)
    print(f"{model} T={T} {bench.FMT} {name} (kcycles per CTA per call): tiles {m[7] * 1e3:.2f}")
    print("  MMA: total %.1f wait_full/xfull %.1f wait_acc_empty %.1f | epilogue wait %.1f work %.1f |"
          " producer wait_empty %.1f" % (m[2], m[0], m[1], m[3], m[4], m[5]))
    print("  expander: wait_full %.1f wait_xempty %.1f stores %.1f fence+arrive %.1f | gather wait %.1f issue %.1f"
          % (m[8], m[9], m[12], m[6], m[10], m[11]))
