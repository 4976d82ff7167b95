"""Diagnostics: two weight objects (tcgen05 path and generic path) on one
context, alternating large prefill batches; per call: ids/gates and output
compared across the two paths and across a repeat of the generic call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_07033_b200 as M  # noqa: E402


def call(ww, x, n):
    xo = torch.empty_like(x)
    ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((n, 2), device="cuda")
    ww.layer_forward(0, x, xo, ids, g)
    torch.cuda.synchronize()
    return xo, ids, g


def main(n, iters):
    d, f = 4096, 14336
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(1, 8, 2, d, f, 2), M.DTYPE_BF16)
    M.set_option("prefill", 0)
    wg = M.Weights(ctx, M.Shape(1, 8, 2, d, f, 2), M.DTYPE_BF16)
    M.set_option("prefill", 1)
    w.random(5)
    wg.random(5)
    for it in range(iters):
        x = torch.randn(n, d, device="cuda")
        og, ig, gg = call(wg, x, n)
        ot, it_, gt = call(w, x, n)
        og2, ig2, gg2 = call(wg, x, n)
        dg, dt, dg2 = (og - x), (ot - x), (og2 - x)
        rel = lambda a, b: float((a - b).abs().max() / b.abs().max())  # noqa: E731
        print(f"it {it}: ids gen==tc {torch.equal(ig, it_)} gen==gen2 {torch.equal(ig, ig2)} | "
              f"gates eq {torch.equal(gg, gt)} | gen vs tc {rel(dg, dt):.2e} gen2 vs tc {rel(dg2, dt):.2e} "
              f"gen vs gen2 {rel(dg, dg2):.2e}", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8192, int(sys.argv[2]) if len(sys.argv) > 2 else 4)
