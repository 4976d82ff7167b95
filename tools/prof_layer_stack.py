"""Drive the single-layer batch-1 path that bench.py's `single_layer_decode`
line times (moe_layer_forward on layer 0 of a multi-layer Mixtral-shaped
stack: one launch of the persistent kernel as a 1-layer stack), for an
`ncu --set full -k regex:decode_stack` capture (tools/round_profile.sh).

    python tools/prof_layer_stack.py [--iters 8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=8)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(2, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
    w.random(0)
    assert w.layer_launches(1) == 1, "the 1-layer stack is not the single-layer path here"
    sp = ctx.stream
    with torch.cuda.stream(torch.cuda.ExternalStream(sp)):
        xs = torch.randn((args.iters, 1, 4096), device="cuda")
        xo = torch.empty((1, 4096), device="cuda")
        ids = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((1, 2), device="cuda")
    torch.cuda.synchronize()
    for i in range(args.iters):
        w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
