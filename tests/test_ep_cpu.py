"""Expert-parallel host logic on CPU, world_size 2 over gloo.

The GPU EP path (capi_orch.cu experts_forward with world > 1) is:
  every rank routes x identically (replicated fp32 router) -> each rank computes
  only the gate-weighted outputs of the experts it owns -> all-reduce(sum) of the
  d-vector delta -> x += delta -> next layer.
These tests check, with the oracle as the expert math, that this decomposition
over the popularity shard map reproduces the single-process model_forward
exactly, and that the shard map is a valid balanced partition.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_map(L, E, world, counts=None):
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    return bench.shard_map(L, E, world, counts)


def _ep_worker(rank, world, port, shape_t, seed, tok_seed, n_tok, counts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O.build(ref=False)
        orc = O.Oracle()
        shape = O.Shape(*shape_t)
        L, E, k = shape.num_layers, shape.experts_per_layer, shape.top_k
        owner = _shard_map(L, E, world, counts)
        w = orc.random_model(shape, seed)  # weights are per-expert; a rank touches only its own
        xs = orc.normal(tok_seed, n_tok * shape.hidden_dim).reshape(n_tok, shape.hidden_dim)
        routes = []
        for t in range(n_tok):
            x = xs[t].copy()
            for l in range(L):
                ids, g, _ = orc.gate_topk(w.router[l], x, k)
                routes.append(list(ids))
                delta = np.zeros_like(x)
                for e, ge in zip(ids, g):
                    if owner[l, e] == rank:
                        wi, wg, wo = w.expert(l, int(e))
                        delta += ge * orc.expert_ffn(wi, wg, wo, x)
                dt = torch.from_numpy(delta)
                dist.all_reduce(dt, op=dist.ReduceOp.SUM)
                x = x + dt.numpy()
            xs[t] = x
        q.put((rank, xs, routes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("skewed", [False, True])
def test_ep_decomposition_matches_single_process(skewed):
    shape_t = (3, 8, 2, 32, 64, 2)
    shape = O.Shape(*shape_t)
    counts = None
    if skewed:  # a popularity profile as profile_from_trace would produce
        rs = np.random.RandomState(1)
        counts = rs.randint(0, 100, size=(3, 8)).astype(np.int64)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ep_worker, args=(r, world, port, shape_t, 5, 6, 3, counts, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (xs, routes)) for r, xs, routes in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = O.Oracle()
    w = orc.random_model(shape, 5)
    toks = orc.normal(6, 3 * 32).reshape(3, 32)
    want, tally, gsum, ids, gates = orc.model_forward(shape, w, toks)
    for r in range(world):
        xs, routes = res[r]
        # both ranks hold the same residual stream and routing
        assert routes == res[0][1]
        np.testing.assert_allclose(xs, want, rtol=0, atol=1e-12)
    assert [list(v) for v in ids.reshape(-1, 2)] == res[0][1]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_map_is_balanced_partition(world):
    rs = np.random.RandomState(world)
    counts = rs.randint(0, 1000, size=(32, 8)).astype(np.int64)
    owner = _shard_map(32, 8, world, counts)
    assert owner.shape == (32, 8)
    assert owner.min() >= 0 and owner.max() < world
    for l in range(32):
        per_rank = np.bincount(owner[l], minlength=world)
        assert (per_rank == 8 // world).all()
        order = sorted(range(8), key=lambda e: (-counts[l, e], e))
        if world > 1:
            assert owner[l, order[0]] != owner[l, order[1]]  # two hottest experts split
    # uniform popularity -> round robin in the reference's (layer, expert) order
    uni = _shard_map(2, 8, world)
    assert list(uni[0]) == [e % world for e in range(8)]


def _replica_worker(rank, world, port, q):
    """EP with a replicated hot expert: each rank plans its share of every
    expert's sorted rows on its own (moe_replica_plan, the device planner's
    host mirror) and computes only those rows (oracle math); the all-reduced
    deltas must equal model_forward, and the ranks' independent plans must
    tile every expert's rows exactly once."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2402_07033_b200 as M

        O.build(ref=False)
        orc = O.Oracle()
        shape = O.Shape(1, 8, 2, 32, 64, 2)
        w = orc.random_model(shape, 7)
        w.router[0][0, :] = 0.5  # with x ~ N(1, 1): expert 0 in every token's top-2
        n = 120
        xs = orc.normal(8, n * 32).reshape(n, 32) + 1.0
        route = [orc.gate_topk(w.router[0], xs[t], 2)[:2] for t in range(n)]
        counts = np.zeros(8, np.int32)
        for ids, _ in route:
            for e in ids:
                counts[e] += 1
        owner = np.arange(8) % world
        holders = (1 << owner).astype(np.uint32)
        holders[int(np.argmax(counts))] = (1 << world) - 1
        # compute-bound cost model with 16-row chunks, so the hot expert splits
        lo, hi, _ = M.replica_plan(counts, holders, world, 1000, 100, 0, 16, rank)
        delta = np.zeros_like(xs)
        for e in range(8):
            rows = [(t, j) for t in range(n) for j in range(2) if route[t][0][j] == e]
            for t, j in rows[lo[e]:hi[e]]:
                wi, wg, wo = w.expert(0, e)
                delta[t] += route[t][1][j] * orc.expert_ffn(wi, wg, wo, xs[t])
        dt = torch.from_numpy(delta)
        dist.all_reduce(dt, op=dist.ReduceOp.SUM)
        plans = [None] * world
        dist.all_gather_object(plans, (lo.tolist(), hi.tolist()))
        q.put((rank, xs + dt.numpy(), plans, counts.tolist(), holders.tolist()))
    finally:
        dist.destroy_process_group()


def test_replicated_expert_split_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = O.Oracle()
    shape = O.Shape(1, 8, 2, 32, 64, 2)
    w = orc.random_model(shape, 7)
    w.router[0][0, :] = 0.5
    want = orc.model_forward(shape, w, orc.normal(8, 120 * 32).reshape(120, 32) + 1.0)[0]
    out, plans, counts, holders = res[0]
    np.testing.assert_allclose(out, want, rtol=0, atol=1e-12)
    np.testing.assert_array_equal(res[1][0], out)
    hot = int(np.argmax(counts))
    assert counts[hot] == 120
    split = [r for r in range(world) if plans[r][1][hot] > plans[r][0][hot]]
    assert len(split) == 2  # the hot expert's rows really are shared
    for e in range(8):  # every expert's rows tiled once, by holders only
        segs = sorted((plans[r][0][e], plans[r][1][e], r) for r in range(world)
                      if plans[r][1][e] > plans[r][0][e])
        pos = 0
        for a, b, r in segs:
            assert a == pos and (holders[e] >> r) & 1
            pos = b
        assert pos == counts[e]
