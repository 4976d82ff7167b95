"""A/B sweep of the grouped prefill kernel's tail-balancing knobs on one box:
max K splits (prefill_splits, read at weights creation) x the eighths of the
experts that take the finest split (pf_late8), 512-token Mixtral layer,
interleaved rounds, median layer time (CUDA events, distinct token batches).

    python tools/sweep_prefill_splits.py [--tokens 512] [--rounds 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cfgs", default="2:3,4:2,4:3,3:3,2:8,4:8,1:0",
                    help="S:late8[:slo[:lag[:cut16]]] (slo = K split of the other experts' downs, 0 = S/2; "
                         "lag = pf_lag, 8 = every down after every up; cut16 = uneven 2-way split point "
                         "in sixteenths of K, small pieces last, 0 = even)")
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    n, d, f, E, k = args.tokens, 4096, 14336, 8, 2
    ctx = M.Ctx(0)
    sp = ctx.stream
    st = torch.cuda.ExternalStream(sp)
    def parse(c):
        v = [int(t) for t in c.split(":")]
        return tuple(v + [0, 8, 0][len(v) - 2:])[:5]

    cfgs = [parse(c) for c in args.cfgs.split(",")]
    ws = {}
    for S in sorted({c[0] for c in cfgs}):
        M.set_option("prefill_splits", S)
        w = M.Weights(ctx, M.Shape(1, E, k, d, f, 2), M.DTYPE_BF16)
        w.random(0)
        w.reserve(n)
        ws[S] = w
    M.set_option("prefill_splits", 2)
    with torch.cuda.stream(st):
        xs = torch.randn((8, n, d), device="cuda")
        xo = torch.empty((n, d), device="cuda")
        ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((n, k), device="cuda")
    torch.cuda.synchronize()
    times = {c: [] for c in cfgs}
    for _ in range(args.rounds):
        for c in cfgs:
            S, late, slo, lag, cut = c
            M.set_option("pf_lag", lag)
            M.set_option("pf_cut16", cut)
            M.set_option("pf_late8", late)
            M.set_option("pf_slo", slo)
            w = ws[S]
            for i in range(3):
                w.layer_forward(0, xs[i % 8], xo, ids, g, stream=sp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(args.iters):
                w.layer_forward(0, xs[i % 8], xo, ids, g, stream=sp)
            e1.record(st)
            torch.cuda.synchronize()
            times[c].append(e0.elapsed_time(e1) / args.iters * 1e3)
    M.set_option("pf_late8", 3)
    M.set_option("pf_slo", 0)
    M.set_option("pf_lag", 8)
    M.set_option("pf_cut16", 0)
    print(json.dumps({f"splits{c[0]}_late{c[1]}_slo{c[2]}_lag{c[3]}_cut{c[4]}": round(float(np.median(v)), 1) for c, v in times.items()},
                     indent=1))


if __name__ == "__main__":
    main()
