"""bench.py — batch-1 MoE decode throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[3]): a 32-layer Mixtral-8x7B-shaped MoE stack
(d=4096, ffn=14336, 8 experts, top-2), bf16 weights (device Philox init,
random), fp32 residual stream, batch 1.  One step = one token through all
32 MoE layers (router -> 2 experts -> combine -> residual, per layer).
At N>1 (torchrun) the experts of every layer are sharded over the ranks by
the popularity placement (expert parallelism; --shard tp: tensor parallelism)
and every layer's partial deltas are combined over NVLink peer memory inside
the persistent kernel (--nccl-combine: ncclAllReduce instead); the metric is
the single token stream's tok/s ("strong" scaling: fixed work).

Reported:
  value     tok/s with the token already in HBM (CUDA events, max over ranks)
  e2e       tok/s through moe_forward_host (pinned host buffers, H2D of the
            token + D2H of the output/routing inside the timed region)
  roofline  the streaming expert kernel alone, timed live with CUDA events
            over the same layers: algorithmic bytes (2 experts x 3 x d x f x 2 B
            = 704,643,072 B per launch) / average launch time vs MEASURED_PEAKS
  cpu_baseline  the reference's own model_forward (oracle/_ref, compiled from
            the reference sources) on a bounded sample on the host cores.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (L, E, k, d, f, dtype)
    "stack32": (32, 8, 2, 4096, 14336, "bf16"),
    "layer": (1, 8, 2, 4096, 14336, "bf16"),
    "x22b": (56, 8, 2, 6144, 16384, "bf16"),
    "tiny": (1, 8, 2, 512, 1792, "f32"),
}
WORKLOAD_NAME = {
    "stack32": "32-layer Mixtral-8x7B-shaped MoE stack decode, batch 1 (BASELINE configs[3])",
    "layer": "single Mixtral-8x7B-shaped MoE layer decode, batch 1 (BASELINE configs[1])",
    "x22b": "56-layer Mixtral-8x22B-shaped MoE stack decode, batch 1 (BASELINE configs[4])",
    "tiny": "tiny MoE layer d=512 f=1792 fp32 decode, batch 1 (BASELINE configs[0])",
}
METRIC = "Mixtral-8x7B MoE decode tok/s (batch 1)"
PREFILL_METRIC = "Mixtral-8x7B MoE layer prefill tok/s (512 tokens, 1 layer)"
PREFILL_WORKLOAD = "Mixtral-8x7B-shaped MoE layer prefill, 512 tokens (BASELINE configs[2])"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(n_gpus):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_map(L, E, world, rank_tokens=None):
    """Expert -> rank map: the reference's popularity ranking (placement.cpp:53-64)
    with LPT assignment per layer (least-loaded rank, ties to lower rank)."""
    owner = np.zeros((L, E), np.int32)
    counts = np.ones((L, E), np.int64) if rank_tokens is None else rank_tokens
    for l in range(L):
        order = sorted(range(E), key=lambda e: (-counts[l, e], e))
        load = [0] * world
        n = [0] * world
        cap = (E + world - 1) // world
        for e in order:
            r = min((r for r in range(world) if n[r] < cap), key=lambda r: (load[r], r))
            owner[l, e] = r
            load[r] += counts[l, e]
            n[r] += 1
    return owner


def replica_map(owner, world, rank_tokens=None, hot=1):
    """[L x E] rank bitmasks of extra expert holders: per
    layer the `hot` most popular experts (reference ranking, placement.cpp:53-64)
    are replicated on every rank; the prefill path then splits their tokens
    over the holders per step (replica_plan.h)."""
    L, E = owner.shape
    counts = np.ones((L, E), np.int64) if rank_tokens is None else rank_tokens
    mask = np.zeros((L, E), np.uint32)
    for l in range(L):
        for e in sorted(range(E), key=lambda e: (-counts[l, e], e))[:hot]:
            mask[l, e] = (1 << world) - 1
    return mask


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2402_07033_b200 as M

    world, rank, local = dist_setup(args.gpus)
    L, E, k, d, f, dt = CONFIGS[args.config]
    if args.layers:  # a reduced stack (e.g. x22b on one GPU: 56 layers need 270 GB)
        L = args.layers
    dtype = M.DTYPE_BF16 if dt == "bf16" else M.DTYPE_F32
    esz = 2 if dt == "bf16" else 4
    if os.environ.get("MOE_B200_BENCH_SAME_GPU") == "1":
        local = 0  # testing only: every rank on GPU 0 (time-sliced; numbers meaningless)
    torch.cuda.set_device(local)
    ctx = M.Ctx(local)
    if world > 1:
        import torch.distributed as dist

        if args.nccl_combine:
            obj = [M.Ctx.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx.init_ep(world, rank, obj[0])  # NCCL all-reduce combine
        else:
            # fused batch-1 combine over NVLink peer memory (no NCCL needed for
            # decode): all-gather the ranks' exchange-window IPC handles and map
            # every peer's window; this also sets the context's (world, rank)
            handles = [None] * world
            dist.all_gather_object(handles, ctx.peer_window(world, d))
            ctx.open_peers(world, rank, handles)
    elif args.force_ep:
        ctx.init_ep(1, 0, M.Ctx.unique_id())  # 1-rank NCCL: the EP code path on one GPU
    shape = M.Shape(L, E, k, d, f, esz)
    owner = shard_map(L, E, world) if world > 1 and args.shard == "ep" else None
    w = M.Weights(ctx, shape, dtype, owner=owner, tp=(world > 1 and args.shard == "tp"))
    w.random(args.seed)
    w.reserve(1)  # all scratch now: nothing allocates (or syncs) inside the timed loop
    stream_ptr = ctx.stream
    stream = torch.cuda.ExternalStream(stream_ptr, device=f"cuda:{local}")

    # token pool resident in HBM (synthetic N(0,1), identical on every rank)
    n_steps = args.warmup + args.steps
    rs = np.random.RandomState(args.seed + 1)
    pool = torch.tensor(rs.randn(n_steps, d).astype(np.float32), device=f"cuda:{local}")
    x = torch.empty((1, d), dtype=torch.float32, device=f"cuda:{local}")
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device=f"cuda:{local}")
    gates = torch.zeros((L, 1, k), dtype=torch.float32, device=f"cuda:{local}")

    def step(i):
        with torch.cuda.stream(stream):
            x.copy_(pool[i:i + 1])
        w.forward(x, ids, gates, stream=stream_ptr)

    # every rank's weights are initialised before the first peer exchange (the
    # in-kernel peer waits are bounded, so a rank still in w.random() must not
    # be waited on)
    torch.cuda.synchronize()
    barrier(world)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        ev0.record(stream)
        for i in range(args.warmup, n_steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1 and not args.nccl_combine:
        ctx.peer_check()  # a peer that never arrived: fail loudly, not a garbage number
    ms = max_over_ranks(ms, world)
    barrier(world)
    ms_per_step = ms / args.steps
    tok_s = 1000.0 / ms_per_step
    launches = w.forward_launches(1) * args.steps

    # ---- roofline of the dominant kernel, live CUDA events ------------------
    # Single GPU: the whole step is ONE launch of decode_stack_kernel (every
    # layer's experts + routing + residual), so it is the dominant kernel:
    # algorithmic bytes = L x (k*3*d*f*esz expert weights + E*d*4 router).
    # The per-layer streaming expert kernel (EP path) is reported beside it.
    peak, peak_src = load_peaks()
    roof = None
    layer_bytes = k * 3 * d * f * esz + E * d * 4
    expert_kernel = None
    if w.expert_path(1) == 1:
        n_rep = max(8, min(64, 2 * L))
        ypart = torch.empty((ctx.sm_count, d), dtype=torch.float32, device=f"cuda:{local}")
        lay_ids = []
        for l in range(L):
            loc = [e for e in range(E) if owner is None or owner[l, e] == rank]
            sel = sorted(loc[:k]) if len(loc) >= k else sorted(loc)
            lay_ids.append(sel + [sel[0]] * (k - len(sel)))
        idt = torch.tensor(lay_ids, dtype=torch.int32, device=f"cuda:{local}")
        gt = torch.full((L, k), 1.0 / k, dtype=torch.float32, device=f"cuda:{local}")
        xk = pool[0:1].clone()
        for r in range(3):
            w.decode_experts_partial(r % L, xk, idt[r % L], gt[r % L], ypart, stream=stream_ptr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for r in range(n_rep):
            w.decode_experts_partial(r % L, xk, idt[r % L], gt[r % L], ypart, stream=stream_ptr)
        e1.record(stream)
        torch.cuda.synchronize()
        kern_ms = e0.elapsed_time(e1) / n_rep
        n_loc = len(set(lay_ids[0]))
        alg = n_loc * 3 * d * w.tp[2] * esz  # ffn rows resident on this rank (tp: f / N)
        ach = alg / (kern_ms * 1e-3) / 1e9
        expert_kernel = {"kernel": "decode_experts_kernel", "achieved": round(ach, 1),
                         "frac": round(ach / peak, 4), "kernel_us": round(kern_ms * 1e3, 2),
                         "alg_bytes_per_launch": alg,
                         # ncu bytes of the single-GPU layer kernel (profiles/); not for a shard
                         "traffic": args.traffic if world == 1 else None}
        del ypart
    if world == 1 and w.forward_launches(1) == 1:
        n_rep = max(10, min(50, args.steps))
        xs = pool[0:1].clone()
        for _ in range(3):
            w.forward(xs, ids, gates, stream=stream_ptr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n_rep):
            w.forward(xs, ids, gates, stream=stream_ptr)
        e1.record(stream)
        torch.cuda.synchronize()
        kern_ms = e0.elapsed_time(e1) / n_rep
        alg = L * layer_bytes
        ach = alg / (kern_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": args.stack_traffic,
                "kernel": "decode_stack_kernel<bf16,2> (one launch per token)",
                "kernel_us": round(kern_ms * 1e3, 2), "alg_bytes_per_launch": alg,
                "alg_bytes_basis": f"{L} layers x ({k} experts x 3 x {d} x {f} x {esz} B + router {E}x{d}x4 B)",
                "peak_source": peak_src, "expert_kernel": expert_kernel}
    elif expert_kernel is not None:
        roof = {"bound": "hbm", "achieved": expert_kernel["achieved"], "peak": peak, "unit": "GB/s",
                "frac": expert_kernel["frac"], "traffic": expert_kernel["traffic"], "kernel": "decode_experts_kernel",
                "kernel_us": expert_kernel["kernel_us"],
                "alg_bytes_per_launch": expert_kernel["alg_bytes_per_launch"], "peak_source": peak_src}
    if roof is not None and world == 1:
        roof["step_frac"] = round(L * layer_bytes / (ms_per_step * 1e-3) / 1e9 / peak, 4)
    if roof is not None:  # also against north_star's nominal 8 TB/s
        roof["frac_vs_nominal_8tbs"] = round(roof["achieved"] / 8000.0, 4)

    # ---- e2e through the host-buffer C-ABI entry point ----------------------
    host_tokens = rs.randn(args.steps + 2, d)
    for i in range(2):
        w.forward_host(host_tokens[i:i + 1])
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(args.steps):
        w.forward_host(host_tokens[2 + i:3 + i])
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world) / args.steps
    e2e = {"value": round(1000.0 / e2e_ms, 3), "unit": "tok/s", "h2d_bytes_per_step": d * 4,
           "d2h_bytes_per_step": d * 4 + L * k * 4 * 2, "ms_per_step": round(e2e_ms, 4)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, w, pool[args.warmup].cpu().numpy().astype(np.float64), L)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(tok_s, 3), "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if dt == "bf16" else "f32", "data": "synthetic (random-init weights, N(0,1) tokens)",
            "config": {"workload": WORKLOAD_NAME[args.config] + (f" [reduced to {L} layers]" if args.layers else ""),
                       "layers": L, "experts": E, "top_k": k,
                       "hidden": d, "ffn": f, "batch": 1,
                       "parallelism": f"{args.shard}{world}" if world > 1 else "single-gpu",
                       "combine": None if world == 1 else
                       ("ncclAllReduce" if args.nccl_combine else "fused peer-memory exchange (NVLink P2P)"),
                       "path": "persistent stack kernel (1 launch/token)" if w.forward_launches(1) == 1
                       else f"per-layer kernels ({w.forward_launches(1)} launches/token, CUDA graph + PDL)",
                       "l2": f"inputs larger than L2: {L * k * 3 * d * f * esz / 1e9:.1f} GB of expert weights streamed per step"},
            "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "roofline": roof,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    w.close()
    ctx.close()


def run_prefill(args):
    """BASELINE configs[2]: one Mixtral-shaped layer, 512-token prefill, bf16,
    on the tcgen05 grouped-GEMM path.  Reports tok/s and both rooflines."""
    import torch

    import paper_2402_07033_b200 as M

    L, E, k, d, f = 1, 8, 2, 4096, 14336
    n = args.prefill_tokens
    torch.cuda.set_device(0)
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(args.seed)
    assert w.expert_path(n) == 3, "tcgen05 prefill path not selected"
    sp = ctx.stream
    stream = torch.cuda.ExternalStream(sp, device="cuda:0")
    n_batches = args.warmup + args.steps
    gen = torch.Generator(device="cuda:0").manual_seed(args.seed + 1)
    with torch.cuda.stream(stream):
        xs = torch.randn((n_batches, n, d), generator=gen, device="cuda:0")
        xo = torch.empty((n, d), device="cuda:0")
        ids = torch.zeros((n, k), dtype=torch.int32, device="cuda:0")
        g = torch.zeros((n, k), dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    for i in range(args.warmup):
        w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        for i in range(args.warmup, n_batches):
            w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    active = len(set(ids.cpu().numpy().ravel().tolist()))
    # live duration of the dominant kernel (the grouped GEMM): CUDA events on
    # the launching stream around each launch, over a separate loop
    w.kernel_timing(True)
    n_k = max(10, min(args.steps, 50))
    for i in range(n_k):
        w.layer_forward(0, xs[args.warmup + i % args.steps], xo, ids, g, stream=sp)
    tot_us, n_launch = w.kernel_timing(False)
    kern_us = tot_us / max(1, n_launch)
    # e2e through the host-buffer entry point: fp64 host tokens -> H2D ->
    # router + grouped GEMM + combine -> D2H of outputs and routing
    rs = np.random.RandomState(args.seed + 2)
    host = [rs.randn(n, d) for _ in range(3)]
    w.forward_host(host[0])
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = max(3, min(args.steps, 30))
    torch.cuda.synchronize()
    ee0.record(stream)
    for i in range(n_e2e):
        w.forward_host(host[1 + i % 2])
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1) / n_e2e
    e2e = {"value": round(n / (e2e_ms * 1e-3), 1), "unit": "tok/s", "h2d_bytes_per_step": n * d * 4,
           "d2h_bytes_per_step": n * d * 4 + n * k * 8, "ms_per_step": round(e2e_ms, 4)}
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O

        if O.reference_available():
            toks = rs.randn(args.cpu_tokens // 3 or 1, d)
            ref, shape, wr = _mixtral_layer_for_reference(d, f, E, k, toks)
            _, secs = ref.time_forward(shape, wr, toks)
            cpu = {"value": round(len(toks) / secs, 4), "unit": "tok/s", "cores": 1, "kind": "reference",
                   "sample": f"{len(toks)} distinct tokens x 1 Mixtral-shaped layer (reference model_forward, "
                             f"fp64, token-major: cost linear in tokens)", "host_cores": os.cpu_count()}
    bytes_ = active * 3 * d * f * 2 + E * d * 4 + n * d * 4 * 2
    # SURVEY 8d per-launch figure of the grouped kernel: the active experts'
    # weights + X in bf16 + Y out in fp32
    kbytes = active * 3 * d * f * 2 + n * d * (2 + 4)
    flops = 2.0 * 3 * d * f * n * k
    peak_bw, src = load_peaks()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    bw = bytes_ / (ms * 1e-3) / 1e9
    tf = flops / (ms * 1e-3) / 1e12
    kbw = kbytes / (kern_us * 1e-6) / 1e9
    ktf = flops / (kern_us * 1e-6) / 1e12
    print(json.dumps({
        "metric": PREFILL_METRIC, "value": round(n / (ms * 1e-3), 1),
        "unit": "tok/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, N(0,1) tokens)",
        "config": {"workload": PREFILL_WORKLOAD,
                   "l2": "inputs larger than L2: 2.8 GB of expert weights streamed per step; token "
                         "batches rotate over steps",
                   "path": "tcgen05/TMEM grouped GEMM (swap-AB), TMA SW128", "active_experts": active},
        "gpu_launches": w.forward_launches(n) * args.steps, "clocks": clk.summary(), "e2e": e2e,
        "cpu_baseline": cpu,
        "roofline": {"bound": "hbm", "achieved": round(kbw, 1), "peak": peak_bw, "unit": "GB/s",
                     "frac": round(kbw / peak_bw, 4), "frac_vs_nominal_8tbs": round(kbw / 8000.0, 4),
                     "traffic": args.prefill_traffic if n == 512 else None,
                     "kernel": "prefill_grouped_kernel (tcgen05 grouped GEMM, one launch per layer)",
                     "kernel_us": round(kern_us, 2), "alg_bytes_per_launch": kbytes,
                     "alg_bytes_basis": f"{active} experts x 3 x {d} x {f} x 2 B + {n} tokens x {d} x (2 + 4) B",
                     "tensor_tflops": round(ktf, 1), "tensor_frac": round(ktf / peaks["bf16_tflops"], 4),
                     "step_achieved": round(bw, 1), "step_frac": round(bw / peak_bw, 4),
                     "step_tensor_tflops": round(tf, 1), "peak_source": src},
    }), flush=True)
    w.close()
    ctx.close()


def _mixtral_layer_for_reference(d, f, E, k, token, seed=0):
    """fp64 weights of one Mixtral-shaped layer for the reference's CPU path:
    a random router and random N(0,1/sqrt(d)) weights for the experts the
    token(s) route to (the others are never touched by model_forward)."""
    import oracle as O

    ref = O.Reference()
    shape = O.Shape(1, E, k, d, f, 2)
    rs = np.random.RandomState(seed)
    router = rs.randn(E, d) / np.sqrt(d)
    routed = set()
    for t in np.atleast_2d(token):
        routed.update(int(e) for e in ref.gate_topk(router, t, k)[0])
    ids = sorted(routed)
    w = O.Weights(shape, experts=ids)
    for e in ids:
        wi, wg, wo = w.expert(0, int(e))
        for m in (wi, wg, wo):
            m[:] = rs.standard_normal(m.shape) / np.sqrt(d)
    w.router[0][:] = router
    return ref, shape, w


def cpu_baseline(args, gw, token, L):
    """Reference model_forward (oracle/_ref) on one Mixtral-shaped layer, a
    bounded sample of tokens, 1 host thread; scaled to the L-layer stack."""
    import oracle as O

    if not O.reference_available():
        return {"value": None, "unit": "tok/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    _, E, k, d, f, _ = CONFIGS[args.config]
    ref, shape, w = _mixtral_layer_for_reference(d, f, E, k, token)
    n = args.cpu_tokens
    toks = np.repeat(token[None], n, axis=0)
    _, secs = ref.time_forward(shape, w, toks)
    per_tok_layer = secs / n
    return {"value": round(1.0 / (per_tok_layer * L), 5), "unit": "tok/s", "cores": 1, "kind": "reference",
            "sample": f"{n} tokens x 1 Mixtral-shaped layer (fp64 reference model_forward, "
                      f"{per_tok_layer * 1e3:.1f} ms/token/layer), scaled to {L} layers",
            "host_cores": os.cpu_count()}


def run_reference(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, compiled
    from /root/reference sources) on all host cores, same metric/config."""
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    if world > 1 and rank != 0:
        return
    import oracle as O

    prefill = args.config == "prefill512"
    L, E, k, d, f, dt = CONFIGS["layer" if prefill else args.config]
    if args.layers:
        L = args.layers
    if not O.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmoe_ref.so not built"}))
        return
    threads = max(1, min(os.cpu_count() or 1, args.ref_threads or (os.cpu_count() or 1)))
    rs = np.random.RandomState(args.seed + 1)
    # each step: every thread pushes one token through one layer of ONE shared
    # reference model (model_forward is reentrant); decode uses
    # one token everywhere, prefill a distinct token per thread (a bounded
    # sample of the 512-token batch: the reference is token-major, its cost
    # is linear in tokens).  tok/s for an L-layer stack = threads / (t*L).
    token = rs.randn(threads if prefill else 1, d)
    ref, shape, w = _mixtral_layer_for_reference(d, f, E, k, token)
    handle = ref.model_create(shape, w)
    del w
    toks = [token[(i if prefill else 0):(i if prefill else 0) + 1] for i in range(threads)]

    def one_step():
        ts = [threading.Thread(target=ref.model_forward_timed, args=(handle, toks[i]))
              for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    ref.model_destroy(handle)
    secs = sum(times)
    tok_s = threads * args.steps / (secs * L)
    if prefill:
        line = {"impl": "reference", "metric": PREFILL_METRIC, "value": round(tok_s, 5), "unit": "tok/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": PREFILL_WORKLOAD, "parallelism": f"cpu x{threads} threads"},
                "cpu_baseline": {"value": round(tok_s, 5), "unit": "tok/s", "cores": threads, "kind": "reference",
                                 "sample": f"{threads} threads x 1 distinct token x 1 Mixtral-shaped layer per step "
                                           f"(reference model_forward, fp64; token-major, linear in tokens)"},
                "e2e": {"value": round(tok_s, 5), "unit": "tok/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    line = {"impl": "reference", "metric": METRIC, "value": round(tok_s, 5), "unit": "tok/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 / tok_s, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME[args.config], "layers": L, "experts": E, "top_k": k,
                       "hidden": d, "ffn": f, "batch": 1, "parallelism": f"cpu x{threads} threads"},
            "cpu_baseline": {"value": round(tok_s, 5), "unit": "tok/s", "cores": threads, "kind": "reference",
                             "sample": f"{threads} threads x 1 token x 1 Mixtral-shaped layer per step "
                                       f"(reference model_forward, fp64), scaled to {L} layers"},
            "e2e": {"value": round(tok_s, 5), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="stack32", choices=sorted(CONFIGS) + ["prefill512"])
    ap.add_argument("--prefill-tokens", type=int, default=512)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-tokens", type=int, default=12)
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layers", type=int, default=0,
                    help="override the config's layer count (per-layer rate of a stack that does not fit)")
    ap.add_argument("--shard", default="ep", choices=["ep", "tp"],
                    help="N>1: expert parallelism (popularity shard map) or tensor parallelism "
                         "(ffn rows of every expert split over the GPUs)")
    ap.add_argument("--nccl-combine", action="store_true",
                    help="N>1: ncclAllReduce instead of the fused peer-memory combine")
    ap.add_argument("--no-stack", action="store_true",
                    help="per-layer 2-kernel graph instead of the persistent stack kernel")
    ap.add_argument("--stack-kernel", type=int, default=0, choices=[0, 1, 2],
                    help="A/B: 1 = two-barrier persistent kernel, 2 = single-barrier fixed-point kernel (default)")
    ap.add_argument("--force-ep", action="store_true",
                    help="testing: 1-rank NCCL communicator (the expert-parallel code path on one GPU)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the decode kernel from an ncu --set full capture")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.stack_traffic = None
    args.prefill_traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if args.traffic is None:
            args.traffic = tj.get("dram_bytes_per_launch")
        args.stack_traffic = tj.get("stack_dram_bytes_per_launch")
        args.prefill_traffic = tj.get("prefill_dram_bytes_per_launch")
    if args.no_stack or args.stack_kernel or args.force_ep:
        import paper_2402_07033_b200 as M

        if args.no_stack:
            M.set_option("stack", 0)
        if args.stack_kernel:
            M.set_option("stack_kernel", args.stack_kernel)
        if args.force_ep:
            M.set_option("force_ep", 1)
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "prefill512":
        run_prefill(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
