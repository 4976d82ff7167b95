"""Per-phase timing of decode_stack3_kernel (stack_kernel=3) from its clock64
stamps (moe_debug_trace_forward).

    python tools/trace_stack3.py [--layers 32] [--reps 3] [--out f.json]

Slots per (layer, CTA):
  consumers: 0 layer start (after reading x_l)   1 first ring stage landed
             2 up phase done (h complete)        3 z partial published (warp 0)
             4 down phase done                   5 partial-y atomics issued
             6 after the grid barrier            7 x_{l+1} in registers
  producer:  8 last W1/W3 copy issued   9 last W2T copy issued
             10 layer l's routing in hand (after the route mbarrier)
  router:    11 layer l+1's routing committed (all z partials seen)
  layer 0:   12/13 and 14/15 = producer (clock64, globaltimer) at start / end
  layer >0:  12 first copy of the layer issued   13 copy number ring+1 issued
             (= the consumers freed the layer's first stage)
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
    ap.add_argument("--kernel", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    M.set_option("stack_kernel", args.kernel)
    ctx = M.Ctx(0)
    L = args.layers
    w = M.Weights(ctx, M.Shape(L, 8, 2, args.d, args.f, 2), M.DTYPE_BF16)
    w.random(0)
    x = 0.1 * torch.randn(1, args.d, device="cuda")
    ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
    for _ in range(2):
        w.forward(x.clone(), ids, g)
    torch.cuda.synchronize()
    res = []
    med = lambda a: float(np.median(a))  # noqa: E731
    for _ in range(args.reps):
        raw = w.debug_trace_forward(x.clone(), ids, g).copy()
        t, ghz = to_ns(raw)
        rows = []
        for l in range(1, L - 1):
            tl, tn = t[l], t[l + 1]
            rows.append({
                "layer_ns": tn[:, 0].min() - tl[:, 0].min(),
                "up_ns": med(tl[:, 2] - tl[:, 1]),
                "down_ns": med(tl[:, 4] - tl[:, 2]),
                "stream_end_spread_ns": tl[:, 4].max() - tl[:, 4].min(),
                "last_z_to_route_committed_ns": med(tl[:, 11] - tl[:, 3].max()),
                "producer_route_wait_ns": med(tn[:, 10] - tl[:, 9]),
                "route_ready_before_down_done_ns": med(tl[:, 4] - tl[:, 11]),
                "issue_done_before_down_done_ns": med(tl[:, 4] - tl[:, 9]),
                "atomics_ns": med(tl[:, 5] - tl[:, 4]),
                "barrier_after_last_ns": tl[:, 6].max() - tl[:, 5].max(),
                "barrier_wait_med_ns": med(tl[:, 6] - tl[:, 5]),
                "x_read_ns": med(tl[:, 7] - tl[:, 6]),
                "next_first_stage_after_start_ns": med(tn[:, 1] - tn[:, 0]),
                "boundary_ns": med(tn[:, 1] - tl[:, 4]),
                "next_first_issue_before_down_done_ns": med(tl[:, 4] - tn[:, 12]),
                "next_ring_refill_after_start_ns": med(tn[:, 13] - tn[:, 0]),
            })
        total = t[L - 1, :, 7].max() - t[0, :, 0].min()
        avg = {k: round(float(np.mean([r[k] for r in rows])), 1) for k in rows[0]}
        res.append({"total_us": round(total / 1e3, 2), "sm_ghz": round(ghz, 3),
                    "per_layer_avg_ns_layers_1_to_L-2": avg})
    print(json.dumps(res[-1], indent=1))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)
        np.save(args.out.replace(".json", "") + "_ns.npy", t.astype(np.float32))


if __name__ == "__main__":
    main()
