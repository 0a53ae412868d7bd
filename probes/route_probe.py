"""Time the routing kernels alone (samoyeds_route) at decode sizes: CUDA-graph replay of R calls."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10725_b200 as P  # noqa: E402

R = 200
for T, E, k in ((64, 8, 2), (64, 64, 6), (64, 64, 8), (256, 64, 6), (4096, 8, 2)):
    lg = torch.randn(T, E, device="cuda")
    P.route(lg, k)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(R):
            P.route(lg, k)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"T={T} E={E} k={k}: {a.elapsed_time(b) / R * 1e3:.2f} us per samoyeds_route")
