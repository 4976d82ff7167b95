"""Race hunt for the fused prefill layer: many random batches (random token
counts, random data, back-to-back launches without host syncs in between)
through the fused path, each compared BIT for bit with the unfused chain on
the same weights; optionally with W linked expert-parallel ranks on one GPU
(streamed home-rank combine) against the unfused peer all-reduce.

    python tools/fused_stress.py [--iters 200] [--world 0|2|4] [--d 1024 --f 2048]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--world", type=int, default=0, help="0: single GPU; 2/4: linked EP ranks")
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--f", type=int, default=2048)
    ap.add_argument("--max-tokens", type=int, default=700)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    rs = np.random.RandomState(args.seed)
    E, k, d, f = 8, 2, args.d, args.f
    s = M.Shape(1, E, k, d, f, 2)
    bad = 0
    if args.world == 0:
        ctx = M.Ctx(0)
        w = M.Weights(ctx, s, M.DTYPE_BF16)
        w.random(args.seed)
        for it in range(args.iters):
            n = int(rs.randint(2, args.max_tokens))
            x = torch.tensor(rs.randn(n, d).astype(np.float32), device="cuda")
            res = []
            for fused in (1, 0):
                M.set_option("prefill_fused", fused)
                xo = torch.empty_like(x)
                ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
                g = torch.zeros((n, k), device="cuda")
                torch.cuda.synchronize()
                w.layer_forward(0, x, xo, ids, g)
                res.append((xo, ids, g))
            torch.cuda.synchronize()
            ok = all(torch.equal(a, b) for a, b in zip(res[0], res[1]))
            bad += not ok
            if not ok:
                print(f"iter {it} n={n}: MISMATCH", flush=True)
        M.set_option("prefill_fused", 1)
    else:
        W = args.world
        ctxs = [M.Ctx(0) for _ in range(W)]
        M.Ctx.link_peers(ctxs, d, max_tokens=args.max_tokens)
        owner = np.array([[e % W for e in range(E)]], np.int32)
        ws = [M.Weights(c, s, M.DTYPE_BF16, owner=owner) for c in ctxs]
        for w in ws:
            w.random(args.seed)
            w.reserve(args.max_tokens)
        for it in range(args.iters):
            n = int(rs.randint(2, args.max_tokens))
            x = torch.tensor(rs.randn(n, d).astype(np.float32), device="cuda")
            torch.cuda.synchronize()
            res = {}
            for fused in (1, 0):
                M.set_option("prefill_fused", fused)
                outs = [torch.empty_like(x) for _ in range(W)]
                ids = [torch.zeros((n, k), dtype=torch.int32, device="cuda") for _ in range(W)]
                gs = [torch.zeros((n, k), device="cuda") for _ in range(W)]
                torch.cuda.synchronize()
                for r in range(W):
                    ws[r].layer_forward(0, x, outs[r], ids[r], gs[r], stream=ctxs[r].stream)
                for c in ctxs:
                    c.synchronize()
                    c.peer_check()
                res[fused] = outs
            ok = all(torch.equal(res[1][r], res[0][0]) for r in range(W))
            bad += not ok
            if not ok:
                print(f"iter {it} n={n}: MISMATCH", flush=True)
        M.set_option("prefill_fused", 1)
    print(json.dumps({"world": args.world, "iters": args.iters, "mismatches": bad}))


if __name__ == "__main__":
    main()
