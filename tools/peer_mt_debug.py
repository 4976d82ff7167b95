"""Diagnostics for the multi-token peer allreduce with W in-process ranks."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # see tests/conftest.py

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_07033_b200 as M  # noqa: E402


def run(world, order, n=5, d=48, f=96):
    s = M.Shape(1, 8, 2, d, f, 4)
    ctxs = [M.Ctx(0) for _ in range(world)]
    M.Ctx.link_peers(ctxs, d, max_tokens=n)
    ws = [M.Weights(c, s, M.DTYPE_F32, tp=True) for c in ctxs]
    for w in ws:
        w.random(13)
        w.reserve(n)
    x = torch.randn(n, d, device="cuda")
    outs = [torch.empty_like(x) for _ in range(world)]
    ids = [torch.zeros((n, 2), dtype=torch.int32, device="cuda") for _ in range(world)]
    g = [torch.zeros((n, 2), device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for r in order:
        ws[r].layer_forward(0, x, outs[r], ids[r], g[r], stream=ctxs[r].stream)
    errs = []
    for c in ctxs:
        c.synchronize()
        try:
            c.peer_check()
            errs.append(0)
        except M.MoeError:
            errs.append(1)
    same = [torch.equal(outs[r], outs[0]) for r in range(world)]
    print(f"world {world} order {order}: err {errs} same-as-rank0 {same}", flush=True)


if __name__ == "__main__":
    run(2, [0, 1])
    run(3, [0, 1, 2])
    run(4, [0, 1, 2, 3])
    run(4, [3, 2, 1, 0])
