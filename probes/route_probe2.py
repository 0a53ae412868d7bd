"""samoyeds_route alone at small T (CUDA-graph replay of R calls): 1..64 tokens."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10725_b200 as P  # noqa: E402

R = 200
for T, E, k in ((8, 64, 6), (16, 64, 6), (32, 64, 6), (32, 8, 2), (48, 64, 6), (64, 64, 6)):
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
    print(f"T={T} E={E} k={k}: {a.elapsed_time(b) * 1e3 / R:.2f} us per samoyeds_route")
