"""How often the next layer's experts are predictable from R_{l+1} x_l (the
speculative-prefetch experiment of DESIGN.md §5, rejected).

    python tools/route_predictability.py
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2402_07033_b200 as M
ctx = M.Ctx(0)
L = 32
w = M.Weights(ctx, M.Shape(L, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
w.random(0)
R = np.stack([w.download_router(l) for l in range(L)])  # [L][E][d]
hits = {0: 0, 1: 0, 2: 0}; tot = 0
for tok in range(20):
    x = torch.randn(1, 4096, device="cuda")
    xs = [x.cpu().numpy()[0].astype(np.float64)]
    ids_all = []
    cur = x
    for l in range(L):
        out = torch.empty_like(cur)
        ids = torch.zeros((1, 2), dtype=torch.int32, device="cuda"); g = torch.zeros((1, 2), device="cuda")
        w.layer_forward(l, cur, out, ids, g)
        torch.cuda.synchronize()
        ids_all.append(sorted(ids.cpu().numpy()[0].tolist()))
        cur = out
        xs.append(out.cpu().numpy()[0].astype(np.float64))
    for l in range(L - 1):
        pred = np.argsort(-(R[l + 1] @ xs[l]))[:2]   # predict layer l+1 routing from x_l
        n = len(set(pred.tolist()) & set(ids_all[l + 1]))
        hits[n] += 1; tot += 1
print("predict layer l+1 top-2 from R_{l+1} x_l:", {k: round(v / tot, 3) for k, v in hits.items()})
print("expected experts correct per layer:", round((hits[1] + 2 * hits[2]) / (2 * tot), 3))
