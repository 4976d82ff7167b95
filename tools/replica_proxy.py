"""Single-GPU proxy for replicated hot experts in N-GPU expert-parallel
prefill (replica_plan.h).

    python tools/replica_proxy.py [--world 2 4] [--tokens 2048 8192] [--reps 20]

One Mixtral-shaped layer whose router puts expert 0 in every token's top-2
(a hot expert).  Each rank of a W-way expert-parallel model is built on this
GPU in turn as a virtual rank (moe_ctx_set_virtual_rank: no exchange), once
with the plain shard map and once with the hot expert replicated on every
rank (bench.replica_map), and its layer time is measured with CUDA events.
The max over ranks is the N-GPU layer time minus the combine; the planner's
predicted makespan (moe_replica_plan) is printed beside it.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--tokens", type=int, nargs="+", default=[2048, 8192])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2402_07033_b200 as M

    L, E, k, d, f = 1, 8, 2, 4096, 14336
    shape = M.Shape(L, E, k, d, f, 2)
    base = M.Ctx(0)
    full = M.Weights(base, shape, M.DTYPE_BF16)
    full.random(0)
    router = full.download_router(0)
    router[0, :] = 0.05
    full.upload_router(0, router)

    def time_layer(w, ctx, x):
        n = x.shape[0]
        s = torch.cuda.ExternalStream(ctx.stream)
        with torch.cuda.stream(s):
            out = torch.empty_like(x)
            ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
            g = torch.zeros((n, k), device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):
            w.layer_forward(0, x, out, ids, g, stream=ctx.stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.reps):
            w.layer_forward(0, x, out, ids, g, stream=ctx.stream)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.reps, ids

    for n in args.tokens:
        x = torch.randn(n, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) + 1.0
        ms_full, ids = time_layer(full, base, x)
        counts = np.bincount(ids.cpu().numpy().ravel(), minlength=E).astype(np.int32)
        for world in args.world:
            owner = bench.shard_map(L, E, world)
            row = {"tokens": n, "world": world, "counts": counts.tolist(),
                   "single_gpu_ms": round(ms_full, 4)}
            for name, mask in (("plain", None), ("replicated", bench.replica_map(owner, world))):
                per_rank = []
                for r in range(world):
                    ctx = M.Ctx(0)
                    ctx.set_virtual_rank(world, r)
                    w = M.Weights(ctx, shape, M.DTYPE_BF16, owner=owner, replicas=mask)
                    w.random(0)
                    w.upload_router(0, router)
                    w.reserve(n)
                    ms, _ = time_layer(w, ctx, x)
                    per_rank.append(round(ms, 4))
                    if r == 0:
                        cost = w.replica_cost
                    w.close()
                    ctx.close()
                holders = (1 << owner[0]).astype(np.uint32)
                if mask is not None:
                    holders |= mask[0]
                _, _, mk = M.replica_plan(counts, holders, world, *cost, 256, 0)
                row[name] = {"rank_ms": per_rank, "max_ms": max(per_rank),
                             "plan_makespan_ms": round(mk / 1e9, 4)}
            row["speedup"] = round(row["plain"]["max_ms"] / row["replicated"]["max_ms"], 3)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
