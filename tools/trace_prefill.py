"""Per-tile timeline of the persistent grouped prefill kernel.

    python tools/trace_prefill.py [--tokens 512] [--reps 3]

Sets the library's trace path (moe_debug_set_trace_path; the library dumps [CTA][tile][4] globaltimer stamps
per launch: tile|N<<32, producer got the tile, MMA issued its last MMA,
epilogue done) and summarises: per tile kind the producer-to-producer
interval (the SM's streaming time per tile), the epilogue lag behind the
last MMA, and the CTA end-time spread (tail).
"""
import argparse
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--opt", action="append", default=[], help="library debug option name=value")
    args = ap.parse_args()
    path = os.path.join(tempfile.mkdtemp(), "pf_trace.bin")
    import torch

    import paper_2402_07033_b200 as M

    n, d, f, E, k = args.tokens, 4096, 14336, 8, 2
    for o in args.opt:
        name, val = o.split("=")
        M.set_option(name, int(val))
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(1, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(0)
    sp = ctx.stream
    s = torch.cuda.ExternalStream(sp)
    with torch.cuda.stream(s):
        xs = torch.randn((args.reps + 2, n, d), device="cuda")
        xo = torch.empty((n, d), device="cuda")
        ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((n, k), device="cuda")
    torch.cuda.synchronize()
    for i in range(2):
        w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
    torch.cuda.synchronize()
    M.set_trace_path(path)
    for i in range(args.reps):
        w.layer_forward(0, xs[2 + i], xo, ids, g, stream=sp)
    torch.cuda.synchronize()
    M.set_trace_path(None)
    raw = open(path, "rb").read()
    off = 0
    n_ft, n_dt = f // 128, d // 128
    counts = np.bincount(ids.cpu().numpy().ravel(), minlength=E)
    print(f"tokens per expert: {counts.tolist()}")
    while off < len(raw):
        G, cap, _, _ = np.frombuffer(raw, np.int32, 4, off)
        off += 16
        tr = np.frombuffer(raw, np.uint64, G * cap * 4, off).reshape(G, cap, 4).astype(np.float64)
        off += G * cap * 4 * 8
        valid = tr[:, :, 1] > 0
        t0 = tr[:, :, 1][valid].min()
        tend = tr[:, :, 3][valid].max()
        ends = np.array([tr[c, valid[c], 3].max() - t0 for c in range(G) if valid[c].any()])
        starts = np.array([tr[c, 0, 1] - t0 for c in range(G) if valid[c].any()])
        kinds = {"up<=128": [], "up>128": [], "down": []}
        lag = {"up<=128": [], "up>128": [], "down": []}
        for c in range(G):
            nt = int(valid[c].sum())
            for i in range(nt):
                word = int(tr[c, i, 0])
                N = (word >> 32) & 0xffff
                kind = "up" if (word >> 48) & 1 else "down"
                if kind == "up":
                    kind = "up<=128" if N <= 128 else "up>128"
                nxt = tr[c, i + 1, 1] if i + 1 < nt else tr[c, i, 3]
                kinds[kind].append((nxt - tr[c, i, 1]) / 1e3)
                lag[kind].append((tr[c, i, 3] - tr[c, i, 2]) / 1e3)
        print(f"kernel span {(tend - t0) / 1e3:.1f} us; CTA start spread {starts.max() / 1e3:.1f} us; "
              f"CTA end p0/p10/p50/p90/p100 " + "/".join(f"{np.percentile(ends, q) / 1e3:.1f}" for q in (0, 10, 50, 90, 100)) + " us")
        for kname in kinds:
            v = np.array(kinds[kname])
            lg = np.array(lag[kname])
            if len(v):
                print(f"  {kname:8s} tiles {len(v):4d}  interval mean {v.mean():6.1f} us (min {v.min():5.1f} max {v.max():6.1f})"
                      f"  epilogue lag after last MMA issue {lg.mean():5.1f} us")


if __name__ == "__main__":
    main()
