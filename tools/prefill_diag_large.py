import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2402_07033_b200 as M
import oracle as O
O.build(ref=False)
orc = O.Oracle()
for n in (4096, 6144, 8192):
    d, f = 4096, 14336
    ctx = M.Ctx(0)
    s = M.Shape(1, 8, 2, d, f, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    M.set_option("prefill", 0)
    wg = M.Weights(ctx, s, M.DTYPE_BF16)
    M.set_option("prefill", 1)
    w.random(5); wg.random(5)
    x = torch.randn(n, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    outs = []
    for ww in (w, wg):
        xo = torch.full_like(x, float("nan"))
        ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda"); g = torch.zeros((n, 2), device="cuda")
        ww.layer_forward(0, x, xo, ids, g)
        torch.cuda.synchronize()
        outs.append((xo.cpu().numpy().astype(np.float64), ids.cpu().numpy(), g.cpu().numpy()))
    xn = x.cpu().numpy().astype(np.float64)
    for name, (o, ids, g) in zip(("tcgen05", "generic"), outs):
        bad = ~np.isfinite(o).all(axis=1)
        print(n, name, "nonfinite rows", int(bad.sum()), "first", np.nonzero(bad)[0][:8].tolist())
    cache = {}
    for t in (0, n // 2, n - 1):
        ids = outs[0][1][t]; g = outs[0][2][t]
        delta = np.zeros(d)
        for e, ge in zip(ids, g):
            if int(e) not in cache: cache[int(e)] = w.download_expert(0, int(e))
            delta += ge * orc.expert_ffn(*cache[int(e)], xn[t])
        for name, (o, _, _) in zip(("tcgen05", "generic"), outs):
            err = np.abs((o[t] - xn[t]) - delta).max() / np.abs(delta).max()
            print(n, name, "token", t, "err vs oracle %.3e" % err)
    w.close(); wg.close(); ctx.close()
