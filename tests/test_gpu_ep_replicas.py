"""Expert parallelism with replicated hot experts, W ranks
linked on ONE GPU (as tests/test_gpu_ep_peers.py).

A router biased so that one expert is in every token's top-2 makes it the
hot expert; it is replicated on every rank (bench.replica_map) and the
device planner (replica_plan.h) splits its sorted rows over the holders each
step.  Checks: the host mirror of the plan really splits the hot expert;
every rank's output is bit-identical; routing equals the unsharded model;
outputs match the unsharded layer within fp32 rounding; the decode path
(owner-only execution) also matches.
"""
import importlib.util
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_07033_b200 as M  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def _hot_router(w, d, E):
    r = w.download_router(0)
    r[0, :] = 0.05  # x ~ N(1, 1): logit 0 ~ 0.05 * d >> the others
    w.upload_router(0, r)
    return r


@pytest.mark.parametrize("world,n_tok", [(2, 2048), (4, 2048), (2, 300)])
def test_replicated_hot_expert(gpu, world, n_tok):
    L, E, k, d, f = 1, 8, 2, 4096, 14336
    s = M.Shape(L, E, k, d, f, 2)
    b = _bench()
    base = M.Ctx(0)
    full = M.Weights(base, s, M.DTYPE_BF16)
    full.random(21)
    router = _hot_router(full, d, E)
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n_tok, d, device="cuda", generator=gen) + 1.0
    want = torch.empty_like(x)
    ids = torch.zeros((n_tok, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((n_tok, k), device="cuda")
    torch.cuda.synchronize()  # inputs from torch's stream; the model runs on base.stream
    full.layer_forward(0, x, want, ids, g, stream=base.stream)
    base.synchronize()
    counts = np.bincount(ids.cpu().numpy().ravel(), minlength=E).astype(np.int32)
    assert counts[0] == n_tok  # the hot expert is in every token's top-2

    owner = b.shard_map(L, E, world)
    mask = b.replica_map(owner, world)
    assert mask[0, 0] == (1 << world) - 1
    ctxs = [M.Ctx(0) for _ in range(world)]
    M.Ctx.link_peers(ctxs, d, max_tokens=n_tok)
    ws = [M.Weights(c, s, M.DTYPE_BF16, owner=owner, replicas=mask) for c in ctxs]
    for w in ws:
        w.random(21)
        w.upload_router(0, router)
        w.reserve(n_tok)
    # the host mirror of the device plan: does the hot expert split?
    holders = (1 << owner[0]).astype(np.uint32) | mask[0]
    wps, rps, pps = ws[0].replica_cost
    parts = [M.replica_plan(counts, holders, world, wps, rps, pps, 256, r) for r in range(world)]
    n_hold = sum(int(p[1][0] > p[0][0]) for p in parts)
    if n_tok >= 2048:
        assert n_hold >= 2, parts
    else:
        assert n_hold == 1  # 300 rows: memory-bound, streaming it twice would not pay
    outs = [torch.empty_like(x) for _ in range(world)]
    idss = [torch.zeros_like(ids) for _ in range(world)]
    gs = [torch.zeros_like(g) for _ in range(world)]
    torch.cuda.synchronize()
    xd = x.double()
    for rep in range(2):
        for r in range(world):
            ws[r].layer_forward(0, x, outs[r], idss[r], gs[r], stream=ctxs[r].stream)
        for c in ctxs:
            c.synchronize()
            c.peer_check()
        for r in range(1, world):
            assert torch.equal(outs[r], outs[0])
        assert torch.equal(idss[0], ids)
        err = float(((outs[0].double() - xd) - (want.double() - xd)).abs().max()
                    / (want.double() - xd).abs().max())
        assert err < 1e-4, err

    # batch 1: every expert runs on its owner only (replicas idle)
    x1 = x[:1].contiguous()
    want1 = torch.empty_like(x1)
    torch.cuda.synchronize()  # inputs from torch's stream; the model runs on base.stream
    full.layer_forward(0, x1, want1, ids[:1], g[:1], stream=base.stream)
    base.synchronize()
    o1 = [torch.empty_like(x1) for _ in range(world)]
    for r in range(world):
        ws[r].layer_forward(0, x1, o1[r], idss[r][:1], gs[r][:1], stream=ctxs[r].stream)
    for c in ctxs:
        c.synchronize()
        c.peer_check()
    d1 = (want1.double() - x1.double()).abs().max()
    err1 = float((o1[0].double() - want1.double()).abs().max() / d1)
    assert err1 < 1e-4, err1
    for w in ws:
        w.close()
    for c in ctxs:
        c.close()
    full.close()
    base.close()


def test_replica_mask_validation(gpu):
    """A mask naming a rank outside the world is rejected; without replicas
    create_ep is plain expert parallelism (the owner holds each expert)."""
    s = M.Shape(2, 8, 2, 256, 512, 2)
    ctx = M.Ctx(0)
    ctx.set_virtual_rank(2, 0)
    owner = np.tile(np.arange(8) % 2, (2, 1)).astype(np.int32)
    bad = np.zeros((2, 8), np.uint32)
    bad[1, 3] = 0b100  # rank 2 of a 2-rank world
    with pytest.raises(M.MoeError):
        M.Weights(ctx, s, M.DTYPE_BF16, owner=owner, replicas=bad)
    plain = M.Weights(ctx, s, M.DTYPE_BF16, owner=owner)
    zero = M.Weights(ctx, s, M.DTYPE_BF16, owner=owner, replicas=np.zeros((2, 8), np.uint32))
    rep = M.Weights(ctx, s, M.DTYPE_BF16, owner=owner, replicas=np.full((2, 8), 0b11, np.uint32))
    assert zero.device_bytes == plain.device_bytes
    assert rep.device_bytes > plain.device_bytes  # every expert resident on rank 0
    for w in (plain, zero, rep):
        w.close()
    ctx.close()


@pytest.mark.parametrize("dtype,n_tok", [(M.DTYPE_BF16, 1500), (M.DTYPE_F32, 40)])
def test_replicas_odd_world_many_experts(gpu, orc, dtype, n_tok):
    """E = 16, top-4, 3 ranks (E not divisible by the world), every expert
    replicated on 2 ranks: bf16 takes the tcgen05 path with the device plan
    (a tiny cost model so that splits happen), fp32 the generic kernels
    (owner-only execution).  Ranks bit-identical, equal to the unsharded
    layer within fp32 rounding."""
    L, E, k, d, f, world = 1, 16, 4, 256, 512, 3
    esz = 2 if dtype == M.DTYPE_BF16 else 4
    s = M.Shape(L, E, k, d, f, esz)
    b = _bench()
    base = M.Ctx(0)
    full = M.Weights(base, s, dtype)
    full.random(31)
    x = torch.randn(n_tok, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(9))
    want = torch.empty_like(x)
    ids = torch.zeros((n_tok, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((n_tok, k), device="cuda")
    torch.cuda.synchronize()  # inputs from torch's stream; the model runs on base.stream
    full.layer_forward(0, x, want, ids, g, stream=base.stream)
    base.synchronize()
    owner = b.shard_map(L, E, world)
    mask = np.zeros((L, E), np.uint32)
    for e in range(E):
        mask[0, e] = (1 << owner[0, e]) | (1 << ((owner[0, e] + 1) % world))
    ctxs = [M.Ctx(0) for _ in range(world)]
    M.Ctx.link_peers(ctxs, d, max_tokens=n_tok)
    ws = [M.Weights(c, s, dtype, owner=owner, replicas=mask) for c in ctxs]
    for w in ws:
        w.random(31)
        w.replica_cost = (1000, 100, 0)  # compute-bound model: split whenever possible
        w.reserve(n_tok)
    outs = [torch.empty_like(x) for _ in range(world)]
    idss = [torch.zeros_like(ids) for _ in range(world)]
    gs = [torch.zeros_like(g) for _ in range(world)]
    torch.cuda.synchronize()
    for r in range(world):
        ws[r].layer_forward(0, x, outs[r], idss[r], gs[r], stream=ctxs[r].stream)
    for c in ctxs:
        c.synchronize()
        c.peer_check()
    for r in range(1, world):
        assert torch.equal(outs[r], outs[0])
    assert torch.equal(idss[0], ids)
    xd = x.double()
    err = float(((outs[0].double() - xd) - (want.double() - xd)).abs().max() / (want.double() - xd).abs().max())
    assert err < 1e-4, err
    # anchored to the oracle: routing and outputs of a token sample on the
    # ranks' device-held weights (each expert downloaded from its owner)
    from _parity import MARGIN, normwise, oracle_deltas, oracle_route

    xh = x.cpu().numpy().astype(np.float64)
    sample = np.arange(0, n_tok, max(1, n_tok // 40))
    oid, og, _, marg = oracle_route(orc, ws[0].download_router(0), xh[sample], k)
    ok = marg > MARGIN
    assert np.array_equal(idss[0].cpu().numpy()[sample][ok], oid[ok])
    delta = oracle_deltas(orc, lambda e: ws[int(owner[0, e])].download_expert(0, e), xh[sample][ok],
                          oid[ok], og[ok])
    got = outs[0].cpu().numpy().astype(np.float64)[sample][ok] - xh[sample][ok]
    err_o = max(normwise(got[i], delta[i]) for i in range(len(delta)))
    assert err_o < (1e-2 if dtype == M.DTYPE_BF16 else 1e-5), err_o
    if dtype == M.DTYPE_BF16:
        counts = np.bincount(ids.cpu().numpy().ravel(), minlength=E).astype(np.int32)
        holders = (1 << owner[0]).astype(np.uint32) | mask[0]
        split = 0
        for e in range(E):
            parts = [M.replica_plan(counts, holders, world, 1000, 100, 0, 256, r) for r in range(world)]
            split += sum(int(p[1][e] > p[0][e]) for p in parts) > 1
        assert split > 0
    for w in ws:
        w.close()
    for c in ctxs:
        c.close()
    full.close()
    base.close()
