"""Minimal batch-1 stack timing (A/B between library builds via MOE_B200_LIB).

    MOE_B200_LIB=path/to/libmoe_b200.so python tools/time_stack.py [--layers 32] [--iters 200]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--iters", type=int, default=200)
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
    torch.cuda.synchronize()

    def step(i):
        with torch.cuda.stream(s):
            x.copy_(pool[i])
        w.forward(x, ids, g, stream=ctx.stream)

    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(args.iters):
        step(5 + i)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    print(f"{os.environ.get('MOE_B200_LIB', 'current')}: {ms:.4f} ms/token  {1000 / ms:.1f} tok/s  "
          f"{ms * 1000 / L:.1f} us/layer")


if __name__ == "__main__":
    main()
