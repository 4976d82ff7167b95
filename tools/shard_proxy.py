"""Single-GPU proxy for one rank of an N-GPU sharded decode (no exchange).

    python tools/shard_proxy.py --config x22b --shard tp --world 2 [--rank 0]

Rank `rank` of a (world)-way expert- (ep) or tensor-parallel (tp) model is
built on this GPU as a virtual rank (moe_ctx_set_virtual_rank: the per-layer
exchange is skipped), so its per-token time is that rank's streaming work
plus launch gaps — the N-GPU step time minus the combine latency.  Used for
configs that do not fit one GPU (Mixtral-8x22B: 56 layers = 270 GB bf16).
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="x22b")
    ap.add_argument("--shard", default="tp", choices=["ep", "tp"])
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--stack", action="store_true",
                    help="persistent one-launch kernel (debug option virtual_stack) instead of per-layer kernels")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2402_07033_b200 as M

    if args.stack:
        M.set_option("virtual_stack", 1)

    L, E, k, d, f, dt = bench.CONFIGS[args.config]
    ctx = M.Ctx(0)
    ctx.set_virtual_rank(args.world, args.rank)
    shape = M.Shape(L, E, k, d, f, 2)
    if args.shard == "tp":
        w = M.Weights(ctx, shape, M.DTYPE_BF16, tp=True)
    else:
        w = M.Weights(ctx, shape, M.DTYPE_BF16, owner=bench.shard_map(L, E, args.world))
    w.random(0)
    s = torch.cuda.ExternalStream(ctx.stream)
    pool = torch.randn(args.steps + 5, 1, d, device="cuda")
    x = torch.empty(1, d, device="cuda")
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, k), device="cuda")

    def step(i):
        with torch.cuda.stream(s):
            x.copy_(pool[i])
        w.forward(x, ids, g, stream=ctx.stream)

    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(args.steps):
        step(5 + i)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    f_loc = w.tp[2]
    # bytes this rank streams per token: tp -> k experts x f/N rows; ep -> its
    # owned experts among the routed ones (measured from the routing record)
    if args.shard == "tp":
        per_tok = L * k * 3 * d * f_loc * 2
    else:
        owner = bench.shard_map(L, E, args.world)
        idn = ids.cpu().numpy()[:, 0, :]
        per_tok = sum(int((owner[l, idn[l]] == args.rank).sum()) for l in range(L)) * 3 * d * f * 2
    print(json.dumps({"config": args.config, "shard": f"{args.shard}{args.world}", "rank": args.rank,
                      "kernel": "stack" if args.stack else "per-layer",
                      "layers": L, "device_gb": round(w.device_bytes / 1e9, 1),
                      "ms_per_token": round(ms, 4), "rank_tok_s": round(1000 / ms, 2),
                      "rank_gb_per_token_last": round(per_tok / 1e9, 3),
                      "rank_gbs_last_token": round(per_tok / (ms * 1e-3) / 1e9, 1),
                      "launches_per_token": w.forward_launches(1)}))


if __name__ == "__main__":
    main()
