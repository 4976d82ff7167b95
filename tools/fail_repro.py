import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2402_07033_b200 as M
n, d, f = 8192, 4096, 14336
ctx = M.Ctx(0)
w = M.Weights(ctx, M.Shape(1, 8, 2, d, f, 2), M.DTYPE_BF16)
M.set_option("prefill", 0)
wg = M.Weights(ctx, M.Shape(1, 8, 2, d, f, 2), M.DTYPE_BF16)
M.set_option("prefill", 1)
w.random(5); wg.random(5)
keep = os.environ.get("KEEP") == "1"
hold = []
for it in range(4):
    x = torch.randn(n, d, device="cuda")
    row = []
    for name in ("gen", "tc"):
        ww = w if name == "tc" else wg
        xo = torch.empty_like(x)
        ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((n, 2), device="cuda")
        ww.layer_forward(0, x, xo, ids, g)
        torch.cuda.synchronize()
        row.append(f"{name}:{float((xo - x).abs().max()):.2f} ids[0]={ids[0].tolist()} g0={g[0].tolist()}")
        if keep: hold.append((xo, ids, g))
    print(it, " | ".join(row), flush=True)
