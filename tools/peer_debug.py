import os, sys, importlib.util
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # see tests/conftest.py
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2402_07033_b200 as M
spec = importlib.util.spec_from_file_location("bench", "/root/repo/bench.py"); b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
world = int(os.environ.get("W", "4")); mode = os.environ.get("MODE", "ep")
L, E, k, d, f = 3, 8, 2, 4096, 14336
M.set_option("stack_grid", 148 // world)
ctxs = [M.Ctx(0) for _ in range(world)]
M.Ctx.link_peers(ctxs, d)
owner = b.shard_map(L, E, world)
s = M.Shape(L, E, k, d, f, 2)
ws = [M.Weights(c, s, M.DTYPE_BF16, owner=owner) if mode == "ep" else M.Weights(c, s, M.DTYPE_BF16, tp=True) for c in ctxs]
for w in ws: w.random(11)
print("launches", [w.forward_launches(1) for w in ws], flush=True)
torch.cuda.synchronize()
x0 = torch.randn(3, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
for t in range(int(os.environ.get("NTOK", "3"))):
    if t == 0:
        xs = [torch.empty(1, d, device="cuda") for _ in range(world)]
        idss = [torch.zeros((L, 1, k), dtype=torch.int32, device="cuda") for _ in range(world)]
        gs = [torch.zeros((L, 1, k), device="cuda") for _ in range(world)]
    for xr in xs:
        xr.copy_(x0[t % 3:t % 3 + 1])
    torch.cuda.synchronize()
    for r in range(world):
        ws[r].forward(xs[r], idss[r], gs[r], stream=ctxs[r].stream)
    errs = []
    for c in ctxs:
        c.synchronize()
        try:
            c.peer_check(); errs.append(0)
        except Exception as e:
            errs.append(1)
    import ctypes as C
    from paper_2402_07033_b200 import capi
    L_ = capi.lib()
    cnt = []
    for c in ctxs:
        buf = (C.c_uint * 4)()
        L_.moe_debug_peer_counters(c.h, buf, 4)
        cnt.append(list(buf))
    print("token", t, "counters(zseq,seq0..2)", cnt, "err flags", errs, "ids", [i[:, 0].cpu().numpy().tolist() for i in idss], "x0", [float(x[0, 0]) for x in xs], flush=True)
