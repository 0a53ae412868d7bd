"""Decode layer call: eager launches vs CUDA-graph replay (same work)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2503_10725_b200 as P  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
d, f, E, k, g = bench.MODELS[model]
dev = torch.device("cuda")
layer = P.MoELayer(P.MoEConfig(E, k, d, f, 0, g, P.Format(*bench.FMT)), bench.build_layer(P, model, dev),
                   max_tokens=T, device=dev)
x = torch.empty(T, d, dtype=torch.int16, device=dev)
P.synth_fill(x, synth.SEED_X, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
lg = torch.empty(T, E, dtype=torch.float32, device=dev)
P.synth_fill(lg, synth.SEED_LOGITS, synth.DIST_NORMAL, float(synth.normal_scale(1.0)))
out = torch.empty(T, d, dtype=torch.float32, device=dev)
K = 200
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        layer(x, lg, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        layer(x, lg, out)
    b.record()
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / K
    ref = out.clone()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        layer(x, lg, out)
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / K
print(f"{model} T={T}: eager {eager * 1e3:.1f} us/call, graph {graph * 1e3:.1f} us/call, "
      f"max |graph - eager| {float((out - ref).abs().max()):.3e}")
