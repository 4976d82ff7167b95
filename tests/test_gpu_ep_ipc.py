"""Multi-PROCESS expert parallelism through CUDA IPC peer windows.

Two processes (one rank each, gloo for the host-side handshake, as
bench.py does under torchrun) map each other's exchange windows with
cudaIpcOpenMemHandle and run a tensor-parallel model whose per-layer
combine goes through those windows.  With one GPU both processes share it,
so their kernels are time-sliced rather than concurrent; the bounded waits
make progress at each slice.  The *_cross_device cases run automatically
when >= 2 GPUs are visible: rank r on GPU r, the exchange over NVLink P2P
(and the NCCL all-reduce path, comm="nccl", over a 2-rank communicator).
Each rank checks its output against the unsharded model computed locally
on its own GPU.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q, kernel, mode, dev=0, comm="peer"):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2402_07033_b200 as M

    torch.cuda.set_device(dev)
    if kernel == "layer":
        M.set_option("stack", 0)  # per-layer kernels + reduce_exchange

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        if kernel == "prefill":  # bf16 tcgen05 layers: the fused EP / TP prefill combine
            L, E, k, d, f, dt, nm = 2, 8, 2, 1024, 2048, M.DTYPE_BF16, 64
        else:
            L, E, k, d, f, dt, nm = 2, 8, 2, 512, 1792, M.DTYPE_F32, 16
        s = M.Shape(L, E, k, d, f, 2 if dt == M.DTYPE_BF16 else 4)
        base = M.Ctx(dev)
        full = M.Weights(base, s, dt)
        full.random(3)
        ctx = M.Ctx(dev)
        if comm == "peer":
            handles = [None] * world
            dist.all_gather_object(handles, ctx.peer_window(world, d, max_tokens=nm))
            ctx.open_peers(world, rank, handles)
        else:  # NCCL all-reduce combine over a world-rank communicator
            uid = [M.Ctx.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.init_ep(world, rank, uid[0])
        if mode == "tp":
            w = M.Weights(ctx, s, dt, tp=True)
        else:
            owner = np.array([[e % world for e in range(E)] for _ in range(L)], np.int32)
            w = M.Weights(ctx, s, dt, owner=owner)
        if comm == "peer" and kernel != "prefill":
            n_l = w.forward_launches(1)
            assert n_l == (1 if kernel == "stack" else 1 + 2 * L), ("launches", n_l)
        w.reserve(1)
        w.random(3)
        gen = torch.Generator(device=f"cuda:{dev}").manual_seed(5)
        x0 = torch.randn(2, d, device="cuda", generator=gen)
        x = torch.empty(1, d, device="cuda")
        ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, 1, k), device="cuda")
        errs = []
        for t in range(2):
            xr = x0[t:t + 1].clone()
            idr = torch.zeros_like(ids)
            gr = torch.zeros_like(g)
            torch.cuda.synchronize()  # xr / idr / gr come from torch's stream; the model runs on base.stream
            full.forward(xr, idr, gr, stream=base.stream)
            base.synchronize()
            x.copy_(x0[t:t + 1])
            torch.cuda.synchronize()
            dist.barrier()
            w.forward(x, ids, g, stream=ctx.stream)
            ctx.synchronize()
            if comm == "peer":
                ctx.peer_check()
            want = (xr - x0[t:t + 1]).double().cpu().numpy()
            got = (x - x0[t:t + 1]).double().cpu().numpy()
            errs.append(float(np.abs(got - want).max() / np.abs(want).max()))
            assert torch.equal(ids, idr), ("ids", t, ids.flatten().tolist(), idr.flatten().tolist())
        # a multi-token (prefill) layer: the multi-token peer combine
        xm = torch.randn(nm, d, device="cuda", generator=torch.Generator(device=f"cuda:{dev}").manual_seed(9))
        wm = torch.empty_like(xm)
        torch.cuda.synchronize()  # (same: inputs on torch's stream)
        full.layer_forward(0, xm, wm, torch.zeros((nm, k), dtype=torch.int32, device="cuda"),
                           torch.zeros((nm, k), device="cuda"), stream=base.stream)
        base.synchronize()
        om = torch.empty_like(xm)
        idm = torch.zeros((nm, k), dtype=torch.int32, device="cuda")
        gm = torch.zeros((nm, k), device="cuda")
        w.reserve(nm)
        if kernel == "prefill":
            assert w.layer_launches(nm) == 3, ("layer launches", w.layer_launches(nm))  # fused: router, grouped, EP combine
        torch.cuda.synchronize()  # inputs made on torch's stream, kernels on ctx.stream
        dist.barrier()
        w.layer_forward(0, xm, om, idm, gm, stream=ctx.stream)
        ctx.synchronize()
        if comm == "peer":
            ctx.peer_check()
        dm_, dw_ = (om - xm).double(), (wm - xm).double()
        errs.append(float((dm_ - dw_).abs().max() / dw_.abs().max()))
        q.put((rank, max(errs), None))
        dist.barrier()
        w.close()
        ctx.close()
        full.close()
        base.close()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        q.put((rank, None, repr(e)))


def _run_two(kernel, mode, cross, comm="peer"):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, kernel, mode, r if cross else 0, comm))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err, exc in res:
        assert exc is None, f"rank {rank}: {exc}"
        assert err < 1e-4, (rank, err)


@pytest.mark.parametrize("kernel,mode", [("layer", "tp"), ("stack", "tp"), ("stack", "ep"), ("prefill", "ep"),
                                         ("prefill", "tp")])
def test_two_process_ipc(kernel, mode):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    _run_two(kernel, mode, cross=False)


@pytest.mark.parametrize("kernel,mode,comm", [("layer", "tp", "peer"), ("stack", "tp", "peer"),
                                              ("stack", "ep", "peer"), ("layer", "ep", "nccl"),
                                              ("prefill", "ep", "peer")])
def test_two_process_cross_device(kernel, mode, comm):
    """Runs only with >= 2 visible GPUs: the NVLink peer exchange (or the
    2-rank NCCL all-reduce) between two real devices."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    _run_two(kernel, mode, cross=True, comm=comm)
