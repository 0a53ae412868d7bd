import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2503_10725_b200 as P
dev16 = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).cuda()
n_sel = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = synth.weight_bf16(41, 128, 256, integer=True)
x = synth.activations_bf16(42, 64, 256, integer=True)
sel = synth.selection(4, 64, n_sel)
sw, status = P.compress(dev16(w), P.Format(1, 2, 32))
got = P.ssmm(sw, dev16(x), torch.from_numpy(sel).cuda())
torch.cuda.synchronize()
print("ok", got.shape)
