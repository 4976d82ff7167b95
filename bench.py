"""bench.py — batch-1 MoE decode throughput on B200 (BASELINE.json metric).

Workload (BASELINE configs[3]): a 32-layer Mixtral-8x7B-shaped MoE stack
(d=4096, ffn=14336, 8 experts, top-2), bf16 weights (device Philox init,
random), fp32 residual stream, batch 1.  One step = one token through all
32 MoE layers (router -> 2 experts -> combine -> residual, per layer).

Tokens are 0.1 * N(0,1): the reference's model_forward has no normalisation
between layers, so with N(0,1) tokens the random-init 32-layer stack's
residual stream grows doubly exponentially and overflows to inf/NaN by
layer ~8 (each layer adds a delta ~ |x|^2).  At 0.1 the stack stays finite
(|x| rms 0.10 -> 0.15 over 32 layers) and its routing is meaningful
(`routing` reports the smallest 2nd-3rd logit margin over the timed tokens).

The default (N=1) line also carries BASELINE configs[1] (one Mixtral layer,
batch-1 decode) and configs[2] (one layer, 512-token prefill on the tcgen05
grouped GEMM) under `extra_configs`, each with its own clocks, roofline and
e2e, measured on layer 0 of the same weights, plus the same 512-token
prefill through all 32 layers (`stack_prefill512`).

At N>1 the experts of every layer are sharded over the ranks (--shard ep:
popularity shard map = expert parallelism; tp: tensor parallelism) and every
layer's partial deltas are combined over NVLink peer memory inside the
persistent kernel; `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.  The metric is the single token stream's
tok/s ("strong" scaling: fixed work).

Reported:
  value     tok/s with the token already in HBM (CUDA events, max over ranks)
  e2e       tok/s through moe_forward_host (fp64 host token, H2D, forward,
            D2H of output + routing inside the timed region)
  roofline  the dominant kernel (the persistent stack kernel, one launch per
            token), timed live with CUDA events on its stream: algorithmic
            bytes per launch / launch time vs MEASURED_PEAKS
  cpu_baseline  the reference's own model_forward (oracle/_ref, compiled from
            the reference sources) on a bounded sample, 1 host core.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
LAYER_METRIC = "Mixtral-8x7B MoE layer decode tok/s (batch 1, 1 layer)"
PREFILL_METRIC = "Mixtral-8x7B MoE layer prefill tok/s (512 tokens, 1 layer)"
PREFILL_WORKLOAD = "Mixtral-8x7B-shaped MoE layer prefill, 512 tokens (BASELINE configs[2])"
STACK_KERNEL_NAME = {1: "decode_stack_kernel", 2: "decode_stack2_kernel", 3: "decode_stack3_kernel"}
# token scale of the multi-layer stacks (see the module docstring)
STACK_TOKEN_SCALE = 0.1


def token_pool(seed: int, n: int, d: int, layers: int) -> np.ndarray:
    """The bench's synthetic tokens: N(0,1) (scaled by STACK_TOKEN_SCALE for
    multi-layer stacks), float32, from RandomState(seed + 1)."""
    rs = np.random.RandomState(seed + 1)
    x = rs.randn(n, d)
    if layers > 1:
        x *= STACK_TOKEN_SCALE
    return x.astype(np.float32)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


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
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi is streaming (its first sample landed) before the
            # timed region starts
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
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
            # one more sample after the region (a short region may fall
            # between two 50 ms samples)
            n0, t0 = len(self.samples), time.time()
            while len(self.samples) == n0 and time.time() - t0 < 1.0 and self.proc.poll() is None:
                time.sleep(0.01)
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


# ---------------------------------------------------------------------------
# multi-GPU plumbing
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n: int) -> None:
    """`--gpus N` without torchrun: re-run this command with N ranks (one per
    GPU) under torch.distributed.run, and exit with its status."""
    same_gpu = os.environ.get("MOE_B200_BENCH_SAME_GPU") == "1"
    if not same_gpu:
        import torch

        vis = torch.cuda.device_count()
        if vis < n:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {n} needs {n} visible GPUs, found {vis}",
                              "n_gpus": n}), flush=True)
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_setup():
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


def gather_floats(v, world):
    if world <= 1:
        return [v]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, v)
    return out


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
def routing_margins(w, pool, idx, L, E, k, stream_ptr, device):
    """Router logits of every timed token through the bench's own kernel
    (moe_forward_logits: the persistent stack kernel writes the fp32 logits
    its top-k ranked) -> the smallest 2nd-3rd margin / max|logit|."""
    import torch

    idx = list(idx)
    x = torch.empty((1, pool.shape[1]), dtype=torch.float32, device=device)
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device=device)
    g = torch.zeros((L, 1, k), dtype=torch.float32, device=device)
    lg = torch.zeros((len(idx), L, E), dtype=torch.float32, device=device)
    stream = torch.cuda.ExternalStream(stream_ptr, device=device)
    for j, i in enumerate(idx):
        with torch.cuda.stream(stream):
            x.copy_(pool[i:i + 1])
        w.forward_logits(x, ids, g, lg[j], stream=stream_ptr)
    torch.cuda.synchronize()
    a = lg.cpu().numpy().astype(np.float64)
    srt = -np.sort(-a, axis=2)
    margin = (srt[:, :, k - 1] - srt[:, :, k]) / np.maximum(np.abs(a).max(axis=2), 1e-30)
    return {"margin_min": float(margin.min()), "below_1e-5": int((margin < 1e-5).sum()),
            "tokens": len(idx), "layers": L, "finite": bool(np.isfinite(a).all()),
            "source": "moe_forward_logits: the fp32 logits the persistent kernel ranked, every timed token x layer"}


def run_ours(args):
    import torch

    import paper_2402_07033_b200 as M

    world, rank, local = dist_setup()
    L, E, k, d, f, dt = CONFIGS[args.config]
    if args.layers:  # a reduced stack (e.g. x22b on one GPU: 56 layers need 270 GB)
        L = args.layers
    dtype = M.DTYPE_BF16 if dt == "bf16" else M.DTYPE_F32
    esz = 2 if dt == "bf16" else 4
    if os.environ.get("MOE_B200_BENCH_SAME_GPU") == "1":
        local = 0  # testing only: every rank on GPU 0 (time-sliced; numbers meaningless)
    device = f"cuda:{local}"
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
    stream = torch.cuda.ExternalStream(stream_ptr, device=device)

    # token pool resident in HBM (synthetic, identical on every rank)
    n_steps = args.warmup + args.steps
    pool_h = token_pool(args.seed, n_steps, d, L)
    pool = torch.tensor(pool_h, device=device)
    x = torch.empty((1, d), dtype=torch.float32, device=device)
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device=device)
    gates = torch.zeros((L, 1, k), dtype=torch.float32, device=device)

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
    ids_rec = ids.cpu().numpy()  # routing of the last timed token (every rank identical)

    # ---- roofline of the dominant kernel, live CUDA events ------------------
    # The whole step is ONE launch of the persistent stack kernel (every
    # layer's experts + routing + residual; at N>1 with the peer exchange
    # inside), so it is the dominant kernel.  Algorithmic bytes per launch on
    # THIS rank = the expert rows it streams: 1 GPU: L x k x 3 d f esz (+ the
    # router); tp: L x k x 3 d (f/N) esz; ep: the routed experts it owns.
    peaks, peak_src = load_peaks()
    peak = float(peaks["hbm_gbs"])
    router_bytes = E * d * 4
    if world == 1:
        rank_bytes = L * (k * 3 * d * f * esz + router_bytes)
        basis = f"{L} layers x ({k} experts x 3 x {d} x {f} x {esz} B + router {E}x{d}x4 B)"
    elif args.shard == "tp":
        rank_bytes = L * k * 3 * d * w.tp[2] * esz
        basis = f"{L} layers x {k} experts x 3 x {d} x {w.tp[2]} (ffn/{world}) x {esz} B"
    else:
        mine = sum(int(owner[l, e] == rank) for l in range(L) for e in ids_rec[l, 0])
        rank_bytes = mine * 3 * d * f * esz
        basis = f"{mine} routed experts owned by rank {rank} (last token) x 3 x {d} x {f} x {esz} B"
    roof = None
    if w.forward_launches(1) == 1:
        # the timed tokens again, each launch bracketed by its own events
        # (the token copy stays outside; re-running one token in place would
        # feed the stack its own growing output)
        n_rep = max(10, min(50, args.steps))
        for i in range(3):
            step(args.warmup + i)
        torch.cuda.synchronize()
        barrier(world)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_rep)]
        for r, (a0, a1) in enumerate(evs):
            with torch.cuda.stream(stream):
                x.copy_(pool[args.warmup + r % args.steps:args.warmup + r % args.steps + 1])
            a0.record(stream)
            w.forward(x, ids, gates, stream=stream_ptr)
            a1.record(stream)
        torch.cuda.synchronize()
        kern_ms = sum(a0.elapsed_time(a1) for a0, a1 in evs) / n_rep
        ach = rank_bytes / (kern_ms * 1e-3) / 1e9
        per_rank = gather_floats(round(ach, 1), world)
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4),
                # the committed capture is of the 32-layer Mixtral stack
                "traffic": args.stack_traffic if world == 1 and args.config == "stack32" and L == 32 else None,
                "kernel": (f"{STACK_KERNEL_NAME[M.get_option('stack_kernel')]}<bf16,2> (one launch per token)" if world == 1 else
                           "decode_stack_kernel<bf16,2> with in-kernel NVLink exchange (one launch per token per rank)"),
                "kernel_us": round(kern_ms * 1e3, 2), "alg_bytes_per_launch": rank_bytes,
                "alg_bytes_basis": basis, "peak_source": peak_src,
                "frac_vs_nominal_8tbs": round(ach / 8000.0, 4)}
        if world > 1:
            roof["per_rank_achieved"] = per_rank
        else:
            roof["step_frac"] = round(rank_bytes / (ms_per_step * 1e-3) / 1e9 / peak, 4)
            roof["read_ceiling_frac"] = round(ach / 7360.0, 4)  # tools/tma_stream_bench.cu row-chunk stream

    # ---- routing margins of the timed tokens -------------------
    routing = None
    if world == 1 and L > 1:
        try:
            routing = routing_margins(w, pool, range(args.warmup, n_steps), L, E, k, stream_ptr, device)
        except M.MoeError as e:  # e.g. --stack-kernel 1: no logits output
            routing = {"unavailable": str(e)}

    # ---- e2e through the host-buffer C-ABI entry point ----------------------
    host_tokens = token_pool(args.seed + 7, args.steps + 2, d, L).astype(np.float64)
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
           "d2h_bytes_per_step": d * 4 + L * k * 4 * 2, "ms_per_step": round(e2e_ms, 4),
           "api": "moe_forward_host (fp64 host token in, fp64 output + routing out)"}

    extra = None
    if world == 1 and args.config == "stack32" and not args.no_extras:
        extra = {"single_layer_decode": bench_layer(args, w, stream, stream_ptr, device, peaks, peak_src),
                 "prefill512": bench_prefill(args, w, stream, stream_ptr, device, peaks, peak_src),
                 "stack_prefill512": bench_stack_prefill(args, w, stream, stream_ptr, device, peaks, peak_src)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, pool_h[args.warmup].astype(np.float64), L)

    if rank == 0:
        par = f"{args.shard}{world}" if world > 1 else "single-gpu"
        line = {
            "metric": METRIC, "value": round(tok_s, 3), "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if dt == "bf16" else "f32",
            "data": ("synthetic: random-init weights (device Philox N(0,1/sqrt(d))), tokens "
                     + (f"{STACK_TOKEN_SCALE} x N(0,1) (a norm-less random stack overflows from N(0,1))"
                        if L > 1 else "N(0,1)")),
            "config": {"workload": WORKLOAD_NAME[args.config] + (f" [reduced to {L} layers]" if args.layers else ""),
                       "layers": L, "experts": E, "top_k": k,
                       "hidden": d, "ffn": f, "batch": 1, "parallelism": par,
                       "combine": None if world == 1 else
                       ("ncclAllReduce" if args.nccl_combine else "fused peer-memory exchange (NVLink P2P)"),
                       "path": "persistent stack kernel (1 launch/token)" if w.forward_launches(1) == 1
                       else f"per-layer kernels ({w.forward_launches(1)} launches/token, CUDA graph + PDL)",
                       "l2": f"inputs larger than L2: {L * k * 3 * d * f * esz / 1e9:.1f} GB of expert weights streamed per step"},
            "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "roofline": roof,
            "routing": routing, "cpu_baseline": cpu,
        }
        if extra is not None:
            line["extra_configs"] = extra
        print(json.dumps(line), flush=True)
    w.close()
    ctx.close()


def bench_layer(args, w, stream, stream_ptr, device, peaks, peak_src):
    """BASELINE configs[1]: one Mixtral-shaped layer, batch-1 decode (layer 0
    of the bench's weights, N(0,1) tokens) through moe_layer_forward: on one
    GPU one launch of the persistent kernel as a 1-layer stack (routing, both
    projections, combine and residual); otherwise router + streaming expert
    kernel + reduce/residual."""
    import torch

    import paper_2402_07033_b200 as M

    L, E, k, d, f, _ = CONFIGS["layer"]
    n_rep = max(1000, 10 * args.steps)  # >= ~120 ms: spans several clock samples
    toks = torch.tensor(token_pool(args.seed, 8, d, 1), device=device)
    xo = torch.empty((1, d), device=device)
    ids = torch.zeros((1, k), dtype=torch.int32, device=device)
    g = torch.zeros((1, k), device=device)
    launches = w.layer_launches(1)
    for i in range(5):
        w.layer_forward(0, toks[i % 8:i % 8 + 1], xo, ids, g, stream=stream_ptr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for i in range(n_rep):
            w.layer_forward(0, toks[i % 8:i % 8 + 1], xo, ids, g, stream=stream_ptr)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_rep
    alg = k * 3 * d * f * 2
    peak = float(peaks["hbm_gbs"])
    if launches == 1:
        # the dominant (only) kernel: one launch per step, so the back-to-back
        # loop above times it (per-launch event pairs would add ~3 us each)
        kname = f"{STACK_KERNEL_NAME[M.get_option('stack_kernel')]}<bf16,2> as a 1-layer stack (one launch per token)"
        traffic = args.layer_traffic
        kern_ms = ms
        kalg = alg + E * d * 4
        path = "moe_layer_forward: one launch of the persistent kernel as a 1-layer stack"
    else:
        # dominant kernel: the streaming expert kernel, timed alone
        kname = "decode_experts_kernel<bf16,2>"
        traffic = args.traffic
        ypart = torch.empty((w.ctx.sm_count, d), dtype=torch.float32, device=device)
        sel = torch.tensor([1, 5], dtype=torch.int32, device=device)
        gt = torch.full((k,), 0.5, device=device)
        for _ in range(3):
            w.decode_experts_partial(0, toks[0:1], sel, gt, ypart, stream=stream_ptr)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(n_rep):
            w.decode_experts_partial(0, toks[0:1], sel, gt, ypart, stream=stream_ptr)
        e1.record(stream)
        torch.cuda.synchronize()
        kern_ms = e0.elapsed_time(e1) / n_rep
        kalg = alg
        path = "moe_layer_forward: router_topk + decode_experts_kernel (TMA ring) + reduce_residual_kernel"
    ach = kalg / (kern_ms * 1e-3) / 1e9
    # e2e: the host-buffer C-ABI call (moe_forward_host_async on layer 0 +
    # moe_host_wait), one synchronous step per token: token in from pinned
    # host memory, output + routing back
    host = torch.tensor(token_pool(args.seed + 3, 8, d, 1)).pin_memory()
    toks_h = [host[i:i + 1] for i in range(8)]  # the caller's token buffers (views made once)
    out_h = torch.empty((1, d)).pin_memory()
    ids_h = torch.empty((1, k), dtype=torch.int32).pin_memory()
    g_h = torch.empty((1, k)).pin_memory()
    n_e2e = max(200, args.steps)
    for i in range(8):  # warm-up (staging buffers, copy streams)
        w.host_wait(w.forward_host_async(0, toks_h[i % 8], out_h, ids_h, g_h))
    t_start = time.perf_counter()
    for i in range(n_e2e):
        w.host_wait(w.forward_host_async(0, toks_h[i % 8], out_h, ids_h, g_h))
    e2e_ms = (time.perf_counter() - t_start) * 1e3 / n_e2e
    return {"metric": LAYER_METRIC, "value": round(1000.0 / ms, 1), "unit": "tok/s", "ms_per_step": round(ms, 5),
            "steps": n_rep, "higher_is_better": True,
            "config": {"workload": WORKLOAD_NAME["layer"], "path": path, "launches_per_step": launches,
                       "weights": "layer 0 of the bench stack",
                       "l2": "704.6 MB of expert weights per step (> L2)"},
            "clocks": clk.summary(),
            "e2e": {"value": round(1000.0 / e2e_ms, 1), "unit": "tok/s", "h2d_bytes_per_step": d * 4,
                    "d2h_bytes_per_step": d * 4 + 2 * k * 4, "ms_per_step": round(e2e_ms, 5),
                    "api": "moe_forward_host_async(layer 0) + moe_host_wait per token (synchronous steps): "
                           "pinned fp32 token in, output + ids + gates out; host wall clock"},
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "traffic": traffic,
                         "kernel": kname, "kernel_us": round(kern_ms * 1e3, 2),
                         "alg_bytes_per_launch": kalg,
                         "alg_bytes_basis": f"{k} experts x 3 x {d} x {f} x 2 B" + (
                             f" + router {E}x{d}x4 B" if kalg != alg else ""),
                         "peak_source": peak_src,
                         "step_frac": round((alg + E * d * 4) / (ms * 1e-3) / 1e9 / peak, 4)}}


def bench_stack_prefill(args, w, stream, stream_ptr, device, peaks, peak_src):
    """512-token prefill through the whole 32-layer stack (moe_forward,
    the fused prefill layer 32 times): north_star's "prefill tokens/sec" for
    the stack.  Tokens 0.1 x N(0,1) as for decode; 4 token batches rotate."""
    import torch

    import paper_2402_07033_b200 as M

    L, E, k, d, f, _ = CONFIGS["stack32"]
    n = args.prefill_tokens
    w.reserve(n)
    gen = torch.Generator(device=device).manual_seed(args.seed + 7)
    with torch.cuda.stream(stream):
        xs = [STACK_TOKEN_SCALE * torch.randn((n, d), generator=gen, device=device) for _ in range(4)]
        x = torch.empty((n, d), device=device)
        ids = torch.zeros((L, n, k), dtype=torch.int32, device=device)
        g = torch.zeros((L, n, k), dtype=torch.float32, device=device)
    torch.cuda.synchronize()

    def step(i):
        with torch.cuda.stream(stream):
            x.copy_(xs[i % 4])
        w.forward(x, ids, g, stream=stream_ptr)

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    n_steps = 8
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for i in range(n_steps):
            step(i)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_steps
    idn = ids.cpu().numpy()
    active = [len(set(idn[l].ravel().tolist())) for l in range(L)]
    alg = sum(a * 3 * d * f * 2 for a in active) + L * n * d * (2 + 4)
    peak = float(peaks["hbm_gbs"])
    bw = alg / (ms * 1e-3) / 1e9
    return {"metric": "Mixtral-8x7B 32-layer stack prefill tok/s (512 tokens)", "value": round(n / (ms * 1e-3), 1),
            "unit": "tok/s", "ms_per_step": round(ms, 3), "steps": n_steps, "higher_is_better": True,
            "config": {"workload": f"{n}-token prefill through the 32-layer Mixtral-8x7B-shaped stack",
                       "path": f"moe_forward: the fused prefill layer x {L} ({w.forward_launches(n)} launches)",
                       "finite": bool(torch.isfinite(x).all().item())},
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "achieved": round(bw, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(bw / peak, 4), "alg_bytes_per_step": alg,
                         "alg_bytes_basis": "per layer: active experts x 3 x d x f x 2 B + tokens x d x (2 + 4) B",
                         "peak_source": peak_src}}


def bench_prefill(args, w, stream, stream_ptr, device, peaks, peak_src):
    """BASELINE configs[2]: one Mixtral-shaped layer (layer 0 of the given
    weights), 512-token prefill on the tcgen05/TMEM grouped GEMM path."""
    import torch

    import paper_2402_07033_b200 as M

    L, E, k, d, f, _ = CONFIGS["layer"]
    n = args.prefill_tokens
    assert w.expert_path(n) == 3, "tcgen05 prefill path not selected"
    w.reserve(n)
    gen = torch.Generator(device=device).manual_seed(args.seed + 1)
    with torch.cuda.stream(stream):
        xs = [torch.randn((n, d), generator=gen, device=device) for _ in range(8)]
        xo = torch.empty((n, d), device=device)
        ids = torch.zeros((n, k), dtype=torch.int32, device=device)
        g = torch.zeros((n, k), dtype=torch.float32, device=device)
    torch.cuda.synchronize()
    for i in range(max(args.warmup, 8)):
        w.layer_forward(0, xs[i % 8], xo, ids, g, stream=stream_ptr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # >= 100 layers (~50 ms): 20 (10 ms) left the figure to the clock ramp
    # and the box (913k-997k tok/s between boxes for the same build)
    n_steps = max(args.steps, 100)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for i in range(n_steps):
            w.layer_forward(0, xs[i % 8], xo, ids, g, stream=stream_ptr)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_steps
    active = len(set(ids.cpu().numpy().ravel().tolist()))
    # live duration of the dominant kernel (the grouped GEMM): CUDA events on
    # the launching stream around each launch, over a separate loop
    w.kernel_timing(True)
    n_k = max(10, min(n_steps, 50))
    for i in range(n_k):
        w.layer_forward(0, xs[i % 8], xo, ids, g, stream=stream_ptr)
    tot_us, n_launch = w.kernel_timing(False)
    kern_us = tot_us / max(1, n_launch)
    # e2e: the layer call with the 512 tokens copied in from pinned host
    # memory and outputs + routing copied back, stream-ordered
    host = torch.tensor(token_pool(args.seed + 5, n, d, 1)).pin_memory()
    out_h = torch.empty((n, d)).pin_memory()
    ids_h = torch.empty((n, k), dtype=torch.int32).pin_memory()
    # through the pipelined host-buffer API (moe_forward_host_async): each
    # step's H2D of its tokens and D2H of its outputs + routing run on copy
    # streams, overlapping the neighbouring steps' layer; host wall clock from
    # the first enqueue to the last step's results in host memory.  Two
    # distinct pinned input/output sets alternate (independent prefill
    # batches, as in serving).
    hosts = [host, torch.tensor(token_pool(args.seed + 6, n, d, 1)).pin_memory()]
    outs = [out_h, torch.empty((n, d)).pin_memory()]
    ids_hs = [ids_h, torch.empty((n, k), dtype=torch.int32).pin_memory()]
    g_hs = [torch.empty((n, k)).pin_memory() for _ in range(2)]
    n_e2e = max(10, min(n_steps, 100))
    tickets = []
    for i in range(4):  # warm-up of the copy streams / staging slots
        tickets.append(w.forward_host_async(0, hosts[i % 2], outs[i % 2], ids_hs[i % 2], g_hs[i % 2]))
    w.host_wait()
    tickets = []
    t_start = time.perf_counter()
    for i in range(n_e2e):
        if i >= 2:
            w.host_wait(tickets[i - 2])  # this set's previous results have landed
        tickets.append(w.forward_host_async(0, hosts[i % 2], outs[i % 2], ids_hs[i % 2], g_hs[i % 2]))
    w.host_wait()
    e2e_ms = (time.perf_counter() - t_start) * 1e3 / n_e2e
    peak = float(peaks["hbm_gbs"])
    tflops_peak = float(peaks.get("bf16_tflops", 1590.0))
    kbytes = active * 3 * d * f * 2 + n * d * (2 + 4)
    flops = 2.0 * 3 * d * f * n * k
    kbw = kbytes / (kern_us * 1e-6) / 1e9
    bw = (active * 3 * d * f * 2 + E * d * 4 + n * d * 4 * 2) / (ms * 1e-3) / 1e9
    return {"metric": PREFILL_METRIC, "value": round(n / (ms * 1e-3), 1), "unit": "tok/s",
            "ms_per_step": round(ms, 4), "steps": n_steps, "higher_is_better": True,
            "config": {"workload": PREFILL_WORKLOAD, "weights": "layer 0 of the bench weights", "tokens": n,
                       "path": ("router (+ dispatch bases) -> tcgen05/TMEM grouped GEMM (swap-AB) with in-kernel "
                                "row dispatch, combine running alongside (ready queue)"
                                if M.get_option("prefill_fused") else
                                "router_topk_bulk + permute + gather + tcgen05/TMEM grouped GEMM (swap-AB) + combine"),
                       "active_experts": active,
                       "l2": "2.8 GB of expert weights per step (> L2); 8 token batches rotate"},
            "clocks": clk.summary(),
            "e2e": {"value": round(n / (e2e_ms * 1e-3), 1), "unit": "tok/s", "h2d_bytes_per_step": n * d * 4,
                    "d2h_bytes_per_step": n * d * 4 + 2 * n * k * 4, "ms_per_step": round(e2e_ms, 4),
                    "api": "moe_forward_host_async(layer 0): pinned fp32 host tokens in, outputs + ids + gates out; "
                           "copies on their own streams overlap the neighbouring steps; host wall clock"},
            "roofline": {"bound": "hbm", "achieved": round(kbw, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(kbw / peak, 4), "traffic": args.prefill_traffic if n == 512 else None,
                         "kernel": "prefill_grouped_kernel (tcgen05 grouped GEMM, one launch per layer)",
                         "kernel_us": round(kern_us, 2), "alg_bytes_per_launch": kbytes,
                         "alg_bytes_basis": f"{active} experts x 3 x {d} x {f} x 2 B + {n} tokens x {d} x (2 + 4) B",
                         "tensor_tflops": round(flops / (kern_us * 1e-6) / 1e12, 1),
                         "tensor_frac": round(flops / (kern_us * 1e-6) / 1e12 / tflops_peak, 4),
                         "step_achieved": round(bw, 1), "step_frac": round(bw / peak, 4),
                         "step_tensor_tflops": round(flops / (ms * 1e-3) / 1e12, 1), "peak_source": peak_src}}


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


def cpu_baseline(args, token, L):
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
            "mode": "batch-1 latency, 1 thread",
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
    # batch-1 latency of the same reference call on one thread (3 samples)
    lat = [ref.model_forward_timed(handle, toks[0]) for _ in range(3)]
    ref.model_destroy(handle)
    secs = sum(times)
    tok_s = threads * args.steps / (secs * L)
    lat_tok_s = 1.0 / (statistics.median(lat) * L)
    mode = (f"throughput: {threads} concurrent independent model_forward calls (the reference is reentrant, "
            f"SPEC.md:114), 1 token each; batch-1 latency on 1 thread is batch1_latency_tok_s")
    if prefill:
        line = {"impl": "reference", "metric": PREFILL_METRIC, "value": round(tok_s, 5), "unit": "tok/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": PREFILL_WORKLOAD, "parallelism": f"cpu x{threads} threads"},
                "cpu_baseline": {"value": round(tok_s, 5), "unit": "tok/s", "cores": threads, "kind": "reference",
                                 "mode": mode,
                                 "sample": f"{threads} threads x 1 distinct token x 1 Mixtral-shaped layer per step "
                                           f"(reference model_forward, fp64; token-major, linear in tokens)"},
                "batch1_latency_tok_s": round(lat_tok_s, 5),
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
                             "mode": mode,
                             "sample": f"{threads} threads x 1 token x 1 Mixtral-shaped layer per step "
                                       f"(reference model_forward, fp64), scaled to {L} layers"},
            "batch1_latency_tok_s": round(lat_tok_s, 5),
            "e2e": {"value": round(tok_s, 5), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_prefill(args):
    """--config prefill512 alone (BASELINE configs[2]) on a 1-layer model."""
    import torch

    import paper_2402_07033_b200 as M

    L, E, k, d, f, _ = CONFIGS["layer"]
    torch.cuda.set_device(0)
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(args.seed)
    sp = ctx.stream
    stream = torch.cuda.ExternalStream(sp, device="cuda:0")
    peaks, src = load_peaks()
    res = bench_prefill(args, w, stream, sp, "cuda:0", peaks, src)
    res.update({"n_gpus": 1, "warmup": args.warmup, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init weights, N(0,1) tokens)",
                "gpu_launches": w.forward_launches(args.prefill_tokens) * res["steps"]})
    if not args.no_cpu_baseline:
        import oracle as O

        if O.reference_available():
            rs = np.random.RandomState(args.seed + 2)
            toks = rs.randn(max(1, args.cpu_tokens // 3), d)
            ref, shape, wr = _mixtral_layer_for_reference(d, f, E, k, toks)
            _, secs = ref.time_forward(shape, wr, toks)
            res["cpu_baseline"] = {"value": round(len(toks) / secs, 4), "unit": "tok/s", "cores": 1,
                                   "kind": "reference",
                                   "sample": f"{len(toks)} distinct tokens x 1 Mixtral-shaped layer (reference "
                                             f"model_forward, fp64, token-major: cost linear in tokens)",
                                   "host_cores": os.cpu_count()}
    print(json.dumps(res), flush=True)
    w.close()
    ctx.close()


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
    ap.add_argument("--no-extras", action="store_true", help="skip the configs[1]/[2] sub-measurements")
    ap.add_argument("--layers", type=int, default=0,
                    help="override the config's layer count (per-layer rate of a stack that does not fit)")
    ap.add_argument("--shard", default="ep", choices=["ep", "tp"],
                    help="N>1: expert parallelism (popularity shard map) or tensor parallelism "
                         "(ffn rows of every expert split over the GPUs)")
    ap.add_argument("--nccl-combine", action="store_true",
                    help="N>1: ncclAllReduce instead of the fused peer-memory combine")
    ap.add_argument("--no-stack", action="store_true",
                    help="per-layer 2-kernel graph instead of the persistent stack kernel")
    ap.add_argument("--stack-kernel", type=int, default=0, choices=[0, 1, 2, 3],
                    help="A/B: 1 = two-barrier persistent kernel, 2 = single-barrier fixed-point kernel (default)")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=VALUE",
                    help="A/B: set a library debug option (moe_debug_set_option)")
    ap.add_argument("--force-ep", action="store_true",
                    help="testing: 1-rank NCCL communicator (the expert-parallel code path on one GPU)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the decode kernel from an ncu --set full capture")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    if args.impl == "ours" and "WORLD_SIZE" in os.environ and env_int("WORLD_SIZE", 1) != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}"}),
              flush=True)
        sys.exit(2)
    args.stack_traffic = None
    args.prefill_traffic = None
    args.layer_traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if args.traffic is None:
            args.traffic = tj.get("dram_bytes_per_launch")
        args.stack_traffic = tj.get("stack_dram_bytes_per_launch")
        args.prefill_traffic = tj.get("prefill_dram_bytes_per_launch")
        args.layer_traffic = tj.get("layer_stack_dram_bytes_per_launch")
    if args.impl == "ours":
        import paper_2402_07033_b200 as M

        if args.no_stack:
            M.set_option("stack", 0)
        if args.stack_kernel:
            M.set_option("stack_kernel", args.stack_kernel)
        for o in args.opt:  # A/B: any library debug option
            name, val = o.split("=")
            M.set_option(name, int(val))
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
