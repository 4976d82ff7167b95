"""Prefill layer time breakdown, fused vs unfused (CUDA events, distinct token
batches per iteration, 512 tokens on one Mixtral layer):
router alone, permute-free fused layer, fused without PDL (serial launches),
unfused chain, and the grouped kernel alone (moe_debug_kernel_timing).

    python tools/prof_prefill_fused.py [--tokens 512] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    n, d, f, E, k = args.tokens, 4096, 14336, 8, 2
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(1, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(0)
    sp = ctx.stream
    st = torch.cuda.ExternalStream(sp)
    nb = 8
    with torch.cuda.stream(st):
        xs = torch.randn((nb, n, d), device="cuda")
        xo = torch.empty((n, d), device="cuda")
        ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((n, k), device="cuda")
    torch.cuda.synchronize()

    def timeit(fn):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(args.iters):
            fn(i)
        e1.record(st)
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / args.iters * 1e3, 1)

    res = {}
    res["router_us"] = timeit(lambda i: w.router_topk(0, xs[i % nb], ids, g, stream=sp))
    for name, opts in [("fused", {"prefill_fused": 1}), ("fused_nopdl", {"prefill_fused": 1, "no_pdl": 1}),
                       ("unfused", {"prefill_fused": 0}), ("unfused_nopdl", {"prefill_fused": 0, "no_pdl": 1})]:
        for kk, v in opts.items():
            M.set_option(kk, v)
        res[f"{name}_layer_us"] = timeit(lambda i: w.layer_forward(0, xs[i % nb], xo, ids, g, stream=sp))
        w.kernel_timing(True)
        timeit(lambda i: w.layer_forward(0, xs[i % nb], xo, ids, g, stream=sp))
        tot, cnt = w.kernel_timing(False)
        res[f"{name}_grouped_kernel_us"] = round(tot / max(cnt, 1), 1)
        M.set_option("no_pdl", 0)
    M.set_option("prefill_fused", 1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
