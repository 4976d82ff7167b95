"""Per-kernel timing of one Mixtral-shaped prefill layer (torch.profiler /
CUPTI activity records, warm L2 state of a real loop, no replay).

    python tools/prof_prefill.py [--tokens 512] [--iters 50]

Prints, per kernel name, launches per layer and mean us, plus the layer
time from CUDA events.  MOE_B200_<OPTION> environment variables set the
library's debug options (tools/_opts.py: MOE_B200_PREFILL_SPLITS,
MOE_B200_PF_DEBUG, ...).
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=14336)
    ap.add_argument("--no-prof", action="store_true", help="skip torch.profiler (e.g. under ncu)")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2402_07033_b200 as M
    from _opts import from_env

    from_env()
    n, d, f, E, k = args.tokens, args.d, args.f, 8, 2
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(1, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(0)
    sp = ctx.stream
    s = torch.cuda.ExternalStream(sp)
    with torch.cuda.stream(s):
        xs = torch.randn((args.iters + 5, n, d), device="cuda")
        xo = torch.empty((n, d), device="cuda")
        ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((n, k), device="cuda")
    torch.cuda.synchronize()
    for i in range(5):
        w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(args.iters):
        w.layer_forward(0, xs[5 + i], xo, ids, g, stream=sp)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    if args.no_prof:
        print(f"layer {ms * 1e3:.1f} us")
        return
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(args.iters):
            w.layer_forward(0, xs[5 + i], xo, ids, g, stream=sp)
        torch.cuda.synchronize()
    agg = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            agg[ev.name[:60]].append(ev.device_time)
    print(f"layer {ms * 1e3:.1f} us  ({n / (ms * 1e-3):.0f} tok/s)  "
          f"env PREFILL_SPLITS={os.environ.get('MOE_B200_PREFILL_SPLITS')} PF_DEBUG={os.environ.get('MOE_B200_PF_DEBUG')}")
    for name, ts in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {len(ts) / args.iters:5.1f}/layer  mean {sum(ts) / len(ts):8.1f} us  {name}")


if __name__ == "__main__":
    main()
