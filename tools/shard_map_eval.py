"""Expert-parallel shard maps on the bench's 32-layer stack routing:
the popularity LPT map (bench.shard_map / b200::ep_shard_map) vs the
co-selection-aware map (moe_ep_shard_map_coselect), both built from the
device histograms of a calibration batch and scored on held-out tokens.

At batch 1 a layer costs the largest number of a token's k experts held by
one rank (each rank streams its experts' weights; the combine waits for the
slowest), so the score is E[max per-rank multiplicity] — 1 + P(same rank) for
top-2 — and the per-layer streaming bound it implies at the measured copy
peak.  Random-init weights route close to uniformly, so this measures the
mechanism on synthetic routing, not the gain on a trained model's correlated
routing.

    python tools/shard_map_eval.py [--tokens 2048] [--out gpurun_out/shard_map_eval.json]
"""
import argparse
import importlib.util
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2402_07033_b200 as M

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    L, E, k, d, f = args.layers, 8, 2, 4096, 14336
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(args.seed)  # the bench stack's weights
    n = args.tokens
    # the bench's token distribution (bench.token_pool), routed through every layer
    x = torch.tensor(b.token_pool(args.seed, n, d, L), device="cuda")
    ids = torch.zeros((L, n, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, n, k), device="cuda")
    chunk = 512
    for t0 in range(0, n, chunk):
        t1 = min(n, t0 + chunk)
        xi = x[t0:t1].contiguous()
        ii = torch.zeros((L, t1 - t0, k), dtype=torch.int32, device="cuda")
        gi = torch.zeros((L, t1 - t0, k), device="cuda")
        w.forward(xi, ii, gi)
        ids[:, t0:t1] = ii
    torch.cuda.synchronize()
    half = n // 2
    cal = ids[:, :half].contiguous()
    counts = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    pairs = torch.zeros((L, E, E), dtype=torch.int64, device="cuda")
    ctx.routing_histogram(cal, counts)
    ctx.routing_pair_histogram(cal, pairs)
    torch.cuda.synchronize()
    cnt, prs = counts.cpu().numpy(), pairs.cpu().numpy()
    held = ids[:, half:].cpu().numpy()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6540.0}
    expert_bytes = 3 * d * f * 2
    res = {"tokens_calibration": half, "tokens_scored": n - half, "layers": L,
           "note": "random-init weights (close to uniform routing): the mechanism, not a trained model's gain"}
    for world in (2, 4, 8):
        maps = {"popularity_lpt": b.shard_map(L, E, world, rank_tokens=cnt),
                "coselect": M.ep_shard_map_coselect(cnt, prs, world)[0]}
        for name, owner in maps.items():
            mult = np.zeros(held.shape[:2])
            for l in range(L):
                r = owner[l][held[l]]  # [tokens, k] ranks
                mult[l] = np.array([np.bincount(row, minlength=world).max() for row in r])
            streams = float(mult.mean())
            res[f"G{world}_{name}"] = {
                "expert_streams_per_layer": round(streams, 4),
                "p_colocated": round(float((mult > 1).mean()), 4),
                "layer_bound_us": round(streams * expert_bytes / (float(peaks["hbm_gbs"]) * 1e3), 2)}
    print(json.dumps(res, indent=1))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
