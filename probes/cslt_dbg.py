import torch
from torch.sparse import SparseSemiStructuredTensor, to_sparse_semi_structured
torch.manual_seed(0)
m = k = n = 128
w = torch.randint(-2, 3, (m, k), device="cuda").to(torch.bfloat16)
g = w.view(m, k // 4, 4)
idx = g.float().abs().topk(2, dim=-1).indices
mask = torch.zeros_like(g, dtype=torch.bool).scatter_(-1, idx, True)
w = (g * mask).view(m, k)
print("2:4 ok", bool(((w.view(m, k//4, 4) != 0).sum(-1) <= 2).all()))
x = torch.randint(-2, 3, (n, k), device="cuda").to(torch.bfloat16)
xt = x.t().contiguous()
ref = w.float() @ xt.float()
for cut in (False, True):
    SparseSemiStructuredTensor._FORCE_CUTLASS = cut
    ws = to_sparse_semi_structured(w)
    for name, f in (("mm(ws, xt)", lambda: torch.mm(ws, xt)), ("ws @ x.t()", lambda: ws @ x.t()),
                    ("(x @ ws.t()).t()", lambda: (x @ ws.t()).t())):
        try:
            got = f().float()
            print(cut, name, float((got - ref).abs().max()), float((got - ref).norm() / ref.norm()))
        except Exception as e:
            print(cut, name, "ERR", repr(e)[:120])
wc = torch._cslt_compress(w)
for name, b in (("xt", xt), ("x.t()", x.t())):
    got = torch._cslt_sparse_mm(wc, b).float()
    print("cslt", name, tuple(got.shape), float((got - ref).norm() / ref.norm()), float((got.t() - ref).norm() / ref.norm()))
