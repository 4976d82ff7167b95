"""Where the batch-1 step time goes outside the stack kernel.

    python tools/time_gaps.py [--layers 32] [--iters 100]

Times (CUDA events, same stream): forward() back to back on a resident
token; token copy + forward (the bench step); and the copy alone.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--iters", type=int, default=100)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    ctx = M.Ctx(0)
    L = args.layers
    w = M.Weights(ctx, M.Shape(L, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
    w.random(0)
    s = torch.cuda.ExternalStream(ctx.stream)
    pool = torch.randn(args.iters + 5, 1, 4096, device="cuda")
    x = torch.empty(1, 4096, device="cuda")
    ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, 2), device="cuda")
    with torch.cuda.stream(s):
        x.copy_(pool[0])
    for _ in range(5):
        w.forward(x, ids, g, stream=ctx.stream)
    torch.cuda.synchronize()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for i in range(args.iters):
            fn(i)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.iters * 1e3

    def fwd(i):
        w.forward(x, ids, g, stream=ctx.stream)

    def cpy(i):
        with torch.cuda.stream(s):
            x.copy_(pool[i])

    def both(i):
        cpy(i)
        fwd(i)

    for name, fn in (("forward only", fwd), ("copy only", cpy), ("copy + forward", both),
                     ("forward only (again)", fwd)):
        print(f"{name:22s} {timed(fn):9.1f} us/iter")


if __name__ == "__main__":
    main()
