"""A/B of the persistent decode kernels on one weights object:
stack_kernel=1 (two grid barriers per layer, float partial reduction),
stack_kernel=2 (one barrier, fixed-point L2 atomics) and stack_kernel=3 (routing
resolved during the down phase).  Checks routing and
output agreement and run-to-run bit-determinism, then times both.

    python tools/ab_stack.py [--layers 32] [--iters 50]
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
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=14336)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--configs", default="1,2", help="stack_kernel values to time")
    ap.add_argument("--kernels", default="1,2", help="stack_kernel values compared with the first")
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    L, d = args.layers, args.d
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(L, 8, 2, d, args.f, 2), M.DTYPE_BF16)
    w.random(0)
    w.reserve(1)
    sp = ctx.stream
    st = torch.cuda.ExternalStream(sp)
    x0 = args.scale * torch.randn(1, d, device="cuda")  # see bench.py: N(0,1) tokens overflow a norm-less 32-layer stack
    res = {}
    outs = {}
    kerns = [int(k) for k in args.kernels.split(",")]
    for kern in kerns:
        M.set_option("stack_kernel", kern)
        o = []
        for _ in range(3):
            x = x0.clone()
            ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
            g = torch.zeros((L, 1, 2), device="cuda")
            torch.cuda.synchronize()
            w.forward(x, ids, g, stream=sp)
            torch.cuda.synchronize()
            o.append((x.cpu().numpy().copy(), ids.cpu().numpy().copy(), g.cpu().numpy().copy()))
        det = all(np.array_equal(o[0][i], oo[i]) for oo in o[1:] for i in range(3))
        outs[kern] = o[0]
        res[f"k{kern}_deterministic"] = bool(det)
    xin = x0.cpu().numpy()
    x1, i1, g1 = outs[kerns[0]]
    for kern in kerns[1:]:
        x2, i2, g2 = outs[kern]
        tag = f"k{kern}_vs_k{kerns[0]}"
        res[f"{tag}_ids_equal"] = bool(np.array_equal(i1, i2))
        res[f"{tag}_x_bit_equal"] = bool(np.array_equal(x1, x2))
        res[f"{tag}_gates_bit_equal"] = bool(np.array_equal(g1, g2))
        res[f"{tag}_first_ids_diff_layer"] = int(np.argmax((i1 != i2).any(axis=(1, 2)))) if not np.array_equal(i1, i2) else -1
        res[f"{tag}_normwise_delta_err"] = float(np.abs((x2 - xin) - (x1 - xin)).max() / np.abs(x1 - xin).max())
    # timing, alternating
    cfgs = [(int(c),) for c in args.configs.split(",")]
    times = {c: [] for c in cfgs}
    x = x0.clone()
    ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, 2), device="cuda")
    for r in range(args.rounds):
        for cfg in cfgs:
            M.set_option("stack_kernel", cfg[0])
            for _ in range(3):
                w.forward(x, ids, g, stream=sp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.iters):
                w.forward(x, ids, g, stream=sp)
            e1.record(st)
            torch.cuda.synchronize()
            times[cfg].append(e0.elapsed_time(e1) / args.iters)
    for cfg in cfgs:
        ms = float(np.median(times[cfg]))
        tag = "k" + "_".join(str(v) for v in cfg)
        res[f"{tag}_ms"] = round(ms, 4)
        res[f"{tag}_tok_s"] = round(1000 / ms, 2)
        res[f"{tag}_gbs"] = round(L * (2 * 3 * d * args.f * 2 + 8 * d * 4) / (ms * 1e-3) / 1e9, 1)
    # logits of the bench token through the kernels >= 2 (bit-equal expected)
    lgs = {}
    for kern in [k for k in kerns if k >= 2]:
        M.set_option("stack_kernel", kern)
        lg = torch.zeros((L, 8), device="cuda")
        xx = x0.clone()
        w.forward_logits(xx, ids, g, lg, stream=sp)
        torch.cuda.synchronize()
        lgs[kern] = lg.cpu().numpy()
    ks = sorted(lgs)
    res["logits_bit_equal"] = bool(all(np.array_equal(lgs[ks[0]], lgs[k]) for k in ks[1:]))
    lgn = lgs[ks[0]]
    srt = -np.sort(-lgn, axis=1)
    res["routing_margin_min"] = float(((srt[:, 1] - srt[:, 2]) / np.abs(lgn).max(axis=1)).min())
    res["logits_ids_consistent"] = bool(np.array_equal(np.sort(np.argsort(-lgn, kind="stable", axis=1)[:, :2], axis=1),
                                                       ids.cpu().numpy()[:, 0]))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
