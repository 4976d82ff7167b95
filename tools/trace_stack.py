"""Per-phase timing of the persistent stack kernel from %globaltimer stamps.

    python tools/trace_stack.py [--layers 32] [--reps 3]

Stamps per (layer, CTA): 0 layer start, 1 first ring stage landed, 2 stream
done, 3 after grid barrier 1, 4 reduce done, 5 after grid barrier 2,
6 producer released, 7 producer issued last copy (see moe_debug_trace_forward).
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=14336)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    ctx = M.Ctx(0)
    L = args.layers
    w = M.Weights(ctx, M.Shape(L, 8, 2, args.d, args.f, 2), M.DTYPE_BF16)
    w.random(0)
    x = torch.randn(1, args.d, device="cuda")
    ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
    for _ in range(2):
        w.forward(x, ids, g)
    torch.cuda.synchronize()
    res = []
    for _ in range(args.reps):
        tr = w.debug_trace_forward(x, ids, g).astype(np.float64)  # [L][G][8] ns
        t0 = tr[0, :, 0].min()
        rows = []
        for l in range(L):
            t = tr[l]
            start = t[:, 0].min()
            rows.append({
                "layer_ns": (tr[l + 1, :, 0].min() if l + 1 < L else t[:, 5].max()) - start,
                "route_ns": np.median(t[:, 6] - t[:, 0]),
                "first_stage_ns": np.median(t[:, 1] - t[:, 6]),
                "stream_med_ns": np.median(t[:, 2] - t[:, 1]),
                "stream_end_spread_ns": t[:, 2].max() - t[:, 2].min(),
                "barrier1_after_last_ns": t[:, 3].max() - t[:, 2].max(),
                "reduce_ns": np.median(t[:, 4] - t[:, 3]),
                "barrier2_ns": np.median(t[:, 5] - t[:, 4]),
                "issue_done_before_stream_end_ns": np.median(t[:, 2] - t[:, 7]),
                "z_ns": np.median(t[:, 11] - t[:, 2]),
                "route_sum_ns": np.median(t[:, 8] - t[:, 0]),
                "route_bar_ns": np.median(t[:, 9] - t[:, 8]),
                "route_topk_ns": np.median(t[:, 10] - t[:, 9]),
                "route_wake_ns": np.median(t[:, 6] - t[:, 10]),
                "barrier1_after_last_z_ns": t[:, 3].max() - t[:, 11].max(),
            })
        total = tr[L - 1, :, 5].max() - t0
        avg = {k: float(np.mean([r[k] for r in rows[1:]])) for k in rows[0]}
        res.append({"total_us": total / 1e3, "per_layer_avg_ns_excl_l0": avg})
    print(json.dumps(res[-1], indent=1))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
