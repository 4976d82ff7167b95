"""B200 microbenchmark records for the reference's cost model.

    python tools/microbench_records.py [--out records.csv] [--layers 1]

Measures, per Mixtral-8x7B-shaped expert, the four workloads of
cost_model.hpp (MicrobenchRecord) and writes the reference's CSV
(`workload,batch_size,latency_ms,layer`, cost_model.cpp:116-156):

  WeightCopy      one expert's bf16 weights (352 MB) pinned host -> HBM
                  (the paper's CPU->GPU expert fetch)
  ActivationCopy  one fp32 hidden vector (16 KB) host -> device, per direction
  FastExec        one expert at batch 1 on the B200 (streaming decode kernel)
  SlowExec        the reference's CPU expert_ffn (fp64, 1 host core) at batch
                  sizes 1, 2, 3 (the slow device of the paper)

then fits them with the REFERENCE's own load_records_csv + fit (oracle/_ref)
and prints the calibrated CostModel, so the reference simulator can replay
traces with B200 numbers.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADER = "workload,batch_size,latency_ms,layer"


def write_records(records, path):
    """records: iterable of (workload, batch_size, latency_ms, layer)."""
    with open(path, "w") as f:
        f.write(HEADER + "\n")
        for wl, b, ms, layer in records:
            f.write(f"{wl},{int(b)},{float(ms)!r},{int(layer)}\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/b200_records.csv")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nonexpert-ms", type=float, default=2.0)
    args = ap.parse_args()
    import torch

    import oracle as O
    import paper_2402_07033_b200 as M

    d, f = 4096, 14336
    records = []
    # ---- WeightCopy: one expert (W1, W3, W2: 3 x f x d bf16) pinned H2D ----
    nbytes = 3 * d * f * 2
    host = torch.empty(nbytes // 2, dtype=torch.bfloat16).pin_memory()
    dev = torch.empty_like(host, device="cuda")
    s = torch.cuda.Stream()
    for r in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            dev.copy_(host, non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        if r:
            records.append(("WeightCopy", 1, e0.elapsed_time(e1), 0))
    del dev, host
    # ---- ActivationCopy: one fp32 hidden vector, per direction ----
    hx = torch.randn(d).pin_memory()
    dx = torch.empty(d, device="cuda")
    for r in range(args.reps + 1):
        n = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(n):
                dx.copy_(hx, non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        if r:
            records.append(("ActivationCopy", 1, e0.elapsed_time(e1) / n, 0))
    # ---- FastExec: one expert at batch 1 (top_k = 1 layer, streaming kernel) ----
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(1, 8, 1, d, f, 2), M.DTYPE_BF16)
    w.random(0)
    assert w.expert_path(1) == 1
    x = torch.randn(1, d, device="cuda")
    ids = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.ones(1, device="cuda")
    yp = torch.empty((ctx.sm_count, d), device="cuda")
    cs = torch.cuda.ExternalStream(ctx.stream)
    for r in range(args.reps + 1):
        n = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        for i in range(n):
            w.decode_experts_partial(0, x, ids, g, yp, stream=ctx.stream)
        e1.record(cs)
        torch.cuda.synchronize()
        if r:
            records.append(("FastExec", 1, e0.elapsed_time(e1) / n, 0))
    w.close()
    ctx.close()
    # ---- SlowExec: the reference's expert_ffn on the host (fp64, 1 core) ----
    cpu_note = "oracle/_ref not built"
    if O.reference_available():
        ref = O.Reference()
        rs = np.random.RandomState(0)
        wi, wg = (rs.standard_normal((f, d)) / np.sqrt(d) for _ in range(2))
        wo = rs.standard_normal((d, f)) / np.sqrt(d)
        for b in (1, 2, 3):
            xs = rs.randn(b, d)
            t0 = time.perf_counter()
            for t in range(b):
                ref.expert_ffn(wi, wg, wo, xs[t])
            records.append(("SlowExec", b, (time.perf_counter() - t0) * 1e3, 0))
        cpu_note = f"reference expert_ffn, fp64, 1 of {os.cpu_count()} host cores"
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    write_records(records, args.out)
    res = {"records": args.out, "n": len(records), "slow_device": cpu_note}
    if O.reference_available():
        res["fit"] = O.Reference().fit_records(os.path.abspath(args.out), args.nonexpert_ms)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
