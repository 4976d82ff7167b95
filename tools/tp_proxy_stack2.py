"""Single-GPU proxy of one tensor-parallel rank's batch-1 decode step: a
32-layer stack with the ffn dimension divided by N (the rows one TP rank
holds), through the default persistent kernel (decode_stack2).  Its time is
the N-GPU step minus the per-layer NVLink exchange.

    python tools/tp_proxy_stack2.py [--ranks 1 2 4 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    ctx = M.Ctx(0)
    L, E, k, d, f = 32, 8, 2, 4096, 14336
    out = {}
    for n in args.ranks:
        w = M.Weights(ctx, M.Shape(L, E, k, d, f // n, 2), M.DTYPE_BF16)
        w.random(0)
        x0 = 0.1 * torch.randn(1, d, device="cuda")
        ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, 1, k), device="cuda")
        x = x0.clone()
        for _ in range(3):
            x.copy_(x0)
            w.forward(x, ids, g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            x.copy_(x0)
            w.forward(x, ids, g)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        layer_bytes = k * 3 * d * (f // n) * 2
        out[f"tp{n}"] = {"ms_per_token": round(ms, 4), "us_per_layer": round(ms * 1e3 / L, 2),
                         "rank_bytes_per_layer": layer_bytes,
                         "rank_TBps": round(layer_bytes * L / (ms * 1e-3) / 1e12, 3),
                         "tok_s_minus_exchange": round(1000 / ms, 1)}
        w.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
