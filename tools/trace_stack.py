"""Per-phase timing of the persistent stack kernel (moe_debug_trace_forward).

    python tools/trace_stack.py [--layers 32] [--reps 3] [--out f.json]

Stamps are SM clock64 values per (layer, CTA) (slot meanings below); slots
12..15 of layer 0 hold (clock64, globaltimer) pairs at kernel start/end used
to convert cycles to ns and to align CTAs (alignment error ~1 us; intra-CTA
intervals are cycle-exact).
  0 routing start (after the previous layer's barrier 1)   6 producer released
  1 first ring stage landed   2 stream done   11 router partial (z) written
  3 after barrier 1   8 logits summed   9 after CTA barrier   10 top-k committed
  4 residual chunk done   5 after barrier 2   7 producer issued its last copy
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def to_ns(tr):
    """[L][G][16] clock64 -> ns on a common timeline."""
    c0, g0, c1, g1 = (tr[0, :, i].astype(np.float64) for i in (12, 13, 14, 15))
    rate = (c1 - c0) / np.maximum(g1 - g0, 1.0)  # cycles per ns, per CTA
    off = g0 - g0.min()
    out = (tr.astype(np.float64) - c0[None, :, None]) / rate[None, :, None] + off[None, :, None]
    return out, float(np.median(rate))


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
    x = 0.1 * torch.randn(1, args.d, device="cuda")
    ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
    for _ in range(2):
        w.forward(x, ids, g)
    torch.cuda.synchronize()
    res = []
    for _ in range(args.reps):
        raw = w.debug_trace_forward(x, ids, g).copy()
        t, ghz = to_ns(raw)
        med = lambda a: float(np.median(a))  # noqa: E731
        rows = []
        for l in range(1, L - 1):
            tl = t[l]
            rows.append({
                "layer_ns": t[l + 1, :, 0].min() - tl[:, 0].min(),
                "route_sum_ns": med(tl[:, 8] - tl[:, 0]) if l > 0 else 0.0,
                "route_bar_ns": med(tl[:, 9] - tl[:, 8]),
                "route_topk_ns": med(tl[:, 10] - tl[:, 9]),
                "route_topk_again_ns": med(tl[:, 12] - tl[:, 10]),
                "producer_wake_ns": med(t[l + 1, :, 6] - tl[:, 10]),
                "first_stage_after_release_ns": med(tl[:, 1] - tl[:, 6]),
                "stream_ns": med(tl[:, 2] - tl[:, 1]),
                "stream_end_spread_ns": tl[:, 2].max() - tl[:, 2].min(),
                "z_ns": med(tl[:, 11] - tl[:, 2]),
                "barrier1_after_last_ns": tl[:, 3].max() - tl[:, 11].max(),
                "barrier1_wait_med_ns": med(tl[:, 3] - tl[:, 11]),
                "route_plus_reduce_ns": med(tl[:, 4] - tl[:, 3]),
                "barrier2_ns": med(tl[:, 5] - tl[:, 4]),
                "consumer_restart_ns": med(t[l + 1, :, 1] - tl[:, 5]),
                "issue_done_before_stream_end_ns": med(tl[:, 2] - tl[:, 7]),
            })
        total = t[L - 1, :, 5].max() - t[0, :, 0].min()
        avg = {k: round(float(np.mean([r[k] for r in rows])), 1) for k in rows[0]}
        res.append({"total_us": round(total / 1e3, 2), "sm_ghz": round(ghz, 3),
                    "per_layer_avg_ns_layers_1_to_L-2": avg})
    print(json.dumps(res[-1], indent=1))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)
        np.save(args.out.replace(".json", "") + "_raw.npy", raw)


if __name__ == "__main__":
    main()
