"""One layer call at a given T (for ncu captures of the decode kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d, f, E, k, g = bench.MODELS[model]
dev = torch.device("cuda")
layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, g, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                   max_tokens=T, device=dev)
x = torch.empty(T, d, dtype=torch.int16, device=dev)
P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
lg = torch.empty(T, E, dtype=torch.float32, device=dev)
P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
out = torch.empty(T, d, dtype=torch.float32, device=dev)
for _ in range(reps):
    layer(x, lg, out)
torch.cuda.synchronize()
