"""Repeat the tcgen05 prefill against the generic CUDA path on many random
batches (races show up as rare large errors).

    python tools/prefill_stress.py [--iters 30] [--tokens 512]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--tokens", type=int, default=512)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    n, d, f = args.tokens, 4096, 14336
    ctx = M.Ctx(0)
    s = M.Shape(1, 8, 2, d, f, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    M.set_option("prefill", 0)
    wg = M.Weights(ctx, s, M.DTYPE_BF16)
    M.set_option("prefill", 1)
    w.random(5)
    wg.random(5)
    worst, bad = 0.0, 0
    for it in range(args.iters):
        x = torch.randn(n, d, device="cuda")
        outs = []
        for ww in (w, wg):
            xo = torch.empty_like(x)
            ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
            g = torch.zeros((n, 2), device="cuda")
            ww.layer_forward(0, x, xo, ids, g)
            torch.cuda.synchronize()
            outs.append((xo - x).double())
        m0, m1 = float(outs[0].abs().max()), float(outs[1].abs().max())
        if not (np.isfinite(m0) and np.isfinite(m1)) or m1 == 0.0:
            print(f"iter {it}: |delta| max tcgen05 {m0:.3e} generic {m1:.3e}")
        err = float((outs[0] - outs[1]).abs().max() / outs[1].abs().max())
        rows = ((outs[0] - outs[1]).abs().amax(dim=1) > 1e-2 * outs[1].abs().max()).nonzero().flatten()
        worst = max(worst, err)
        if err > 1e-2:
            bad += 1
            print(f"iter {it}: err {err:.3e}, bad rows {rows.tolist()[:16]} ({len(rows)})")
    print(f"{os.environ.get('MOE_B200_LIB', 'current')}: worst {worst:.3e}, bad iterations {bad}/{args.iters}")


if __name__ == "__main__":
    main()
