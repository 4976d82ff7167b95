"""Intra-CTA breakdown of a persistent-kernel trace (tools/trace_stack.py
--out X.json writes X_raw.npy): per-layer phase durations from each CTA's
own clock (cross-CTA alignment is only ~1 us good, intra-CTA is exact).

    python tools/stack_breakdown.py gpurun_out/trace_k2_raw.npy [--ghz 1.9557]
"""
import argparse

import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--ghz", type=float, default=1.9557)
    args = ap.parse_args()
    t = np.load(args.raw).astype(np.float64) / args.ghz
    L, G, _ = t.shape
    med = np.median
    rows = []
    for l in range(2, L - 2):
        tl, tn = t[l], t[l + 1]
        bw = tl[:, 3] - tl[:, 11]
        last = int(np.argmin(bw))          # the last CTA to arrive at the barrier
        lastn = int(np.argmin(tn[:, 3] - tn[:, 11]))
        rows.append(dict(
            period=med(tn[:, 3] - tl[:, 3]),
            barrier_latency=bw.min(), barrier_wait_med=med(bw),
            publish=med(tl[:, 11] - tl[:, 2]),
            x_assembly=med(tl[:, 4] - tl[:, 3]),
            wait_route=med(tl[:, 5] - tl[:, 4]),
            producer_route=med(tn[:, 6] - tl[:, 3]),
            first_stage=med(tn[:, 1] - tn[:, 0]),
            release_to_first=med(tn[:, 1] - tn[:, 6]),
            exit_to_first=med(tn[:, 1] - tl[:, 3]),
            stream_med=med(tn[:, 2] - tn[:, 1]), stream_min=(tn[:, 2] - tn[:, 1]).min(),
            stream_max=(tn[:, 2] - tn[:, 1]).max(),
            crit_exit_to_first=(tn[:, 1] - tl[:, 3])[last],
            crit_stream=(tn[:, 2] - tn[:, 1])[lastn],
            issue_end_before_stream_end=med(tn[:, 2] - tn[:, 7]),
        ))
    for k in rows[0]:
        print("%-30s %8.2f us" % (k, np.mean([r[k] for r in rows]) / 1e3))


if __name__ == "__main__":
    main()
