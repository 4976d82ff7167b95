"""Replica split planner (replica_plan.h) on the CPU.

The planner is the reference scheduler's min-max objective
(scheduler.cpp:97-204: minimise max(slow_sum, fast_sum), ties to the smaller
fast-device cost; greedy order count desc / id asc, scheduler.cpp:154-188)
generalised to G ranks: single-holder experts are fixed load; each
replicated expert, largest first, picks how many of its least-loaded holders
share its rows (chunks dealt by water-filling), scoring a choice by
max(largest load, mean load including the replicated experts still to
place), ties to the smaller largest load, then fewer holders.  The library's host entry point (the same code the
device planner runs) is checked against an independent Python restatement and
against the plan's invariants.
"""
import numpy as np
import pytest

import paper_2402_07033_b200 as M

W_PS = 53_870_000  # Mixtral expert: 3*4096*14336*2 B at 6.54 TB/s, in ps
ROW_PS = 251_658   # 6*4096*14336 flop at 1.4 PFLOP/s, in ps
PART_PS = 0
CHUNK = 256


def py_plan(counts, holders, world, w_ps, row_ps, chunk, part_ps=0):
    """Restatement: returns {rank: {e: (lo, hi)}} and the makespan."""
    E = len(counts)
    order = sorted(range(E), key=lambda e: (-counts[e], e))
    load = [0] * world
    parts = {r: {} for r in range(world)}

    def cost(n):
        return part_ps + max(w_ps, n * row_ps)

    def hold(e):
        return [r for r in range(world) if (holders[e] >> r) & 1]

    rem = 0
    for e in range(E):  # single-holder experts: fixed load
        if counts[e] <= 0 or not hold(e):
            continue
        if len(hold(e)) == 1:
            load[hold(e)[0]] += cost(counts[e])
            parts[hold(e)[0]][e] = (0, counts[e])
        else:
            rem += cost(counts[e])
    for e in order:
        m = counts[e]
        if m <= 0 or len(hold(e)) < 2:
            continue
        cand = sorted(hold(e), key=lambda r: (load[r], r))
        rem -= cost(m)
        nch = -(-m // chunk)
        best = None  # (objective, largest load), chunk counts
        for q in range(1, min(len(cand), nch) + 1):
            cnt = [0] * q
            for _ in range(nch):  # water-filling, ties to the earlier holder
                p = min(range(q), key=lambda p: (load[cand[p]] + cost((cnt[p] + 1) * chunk), p))
                cnt[p] += 1
            new = list(load)
            r0 = 0
            for p in range(q):
                a, b = min(r0, m), min(r0 + cnt[p] * chunk, m)
                r0 += cnt[p] * chunk
                if b > a:
                    new[cand[p]] += cost(b - a)
            obj = (max(max(new), -(-(sum(new) + rem) // world)), max(new))
            if best is None or obj < best[0]:
                best = (obj, cnt)
        r0 = 0
        for p, c in enumerate(best[1]):
            a, b = min(r0, m), min(r0 + c * chunk, m)
            r0 += c * chunk
            if b > a:
                load[cand[p]] += cost(b - a)
                parts[cand[p]][e] = (a, b)
    return parts, max(load)


def lib_plan(counts, holders, world, w_ps=W_PS, row_ps=ROW_PS, chunk=CHUNK, part_ps=PART_PS):
    out = {}
    mk = None
    for r in range(world):
        lo, hi, m = M.replica_plan(counts, holders, world, w_ps, row_ps, part_ps, chunk, r)
        out[r] = {e: (int(lo[e]), int(hi[e])) for e in range(len(counts)) if hi[e] > lo[e]}
        assert mk is None or m == mk  # every rank computes the same plan
        mk = m
    return out, mk


def check_cover(parts, counts, holders, world):
    for e, m in enumerate(counts):
        segs = sorted(parts[r][e] + (r,) for r in range(world) if e in parts[r])
        if m == 0 or holders[e] == 0:
            assert not segs
            continue
        pos = 0
        for a, b, r in segs:
            assert (holders[e] >> r) & 1, "rows on a rank that does not hold the expert"
            assert a == pos and b > a
            assert a % CHUNK == 0
            pos = b
        assert pos == m


@pytest.mark.parametrize("seed", range(40))
def test_plan_matches_restatement(seed):
    rs = np.random.RandomState(seed)
    world = int(rs.choice([1, 2, 3, 4, 8]))
    E = int(rs.choice([2, 8, 16, 64]))
    n_tok = int(rs.choice([1, 64, 512, 2048, 8192]))
    p = rs.dirichlet(np.full(E, 0.3))
    counts = rs.multinomial(n_tok * 2, p).astype(np.int32)
    owner = rs.randint(0, world, E)
    rep = rs.randint(0, 1 << world, E) * (rs.rand(E) < 0.5)
    holders = ((1 << owner) | rep).astype(np.uint32)
    part = int(rs.choice([0, 20_000_000]))
    got, mk = lib_plan(counts, holders, world, part_ps=part)
    want, wmk = py_plan(counts.tolist(), holders.tolist(), world, W_PS, ROW_PS, CHUNK, part)
    assert got == want
    assert mk == wmk
    check_cover(got, counts, holders, world)


def test_no_replicas_is_plain_ep():
    counts = np.array([900, 40, 0, 300, 5, 700, 1, 100], np.int32)
    owner = np.array([0, 1, 2, 3, 0, 1, 2, 3])
    holders = (1 << owner).astype(np.uint32)
    got, _ = lib_plan(counts, holders, 4)
    for e, m in enumerate(counts):
        if m:
            assert got[int(owner[e])][e] == (0, int(m))


def test_memory_bound_expert_is_not_split():
    # 512-token prefill: ~128 rows per expert, weight streaming dominates —
    # a second holder would stream the weights twice for nothing
    counts = np.array([300, 128, 128, 128, 100, 100, 80, 60], np.int32)
    holders = np.full(8, 0b11, np.uint32)
    got, _ = lib_plan(counts, holders, 2)
    for e in range(8):
        assert sum(e in got[r] for r in range(2)) == 1


def test_hot_compute_bound_expert_is_split():
    # one expert takes most of an 8192-token batch: splitting its rows over
    # its holders cuts the makespan
    counts = np.array([12000, 600, 600, 600, 600, 600, 600, 784], np.int32)
    owner = np.array([0, 1, 2, 3, 0, 1, 2, 3])
    no_rep, mk0 = lib_plan(counts, (1 << owner).astype(np.uint32), 4)
    holders = (1 << owner).astype(np.uint32)
    holders[0] = 0b1111
    got, mk = lib_plan(counts, holders, 4)
    assert sum(0 in got[r] for r in range(4)) >= 2
    assert mk < mk0
    check_cover(got, counts, holders, 4)


def test_balanced_compute_bound_split():
    # 2048-token batch, one expert in every token's top-2: splitting it costs
    # no extra total work (compute-bound) and halves the hot rank's load
    counts = np.array([2048, 293, 293, 293, 293, 293, 292, 291], np.int32)
    owner = np.array([0, 1, 0, 1, 0, 1, 0, 1])
    holders = (1 << owner).astype(np.uint32)
    _, mk0 = lib_plan(counts, holders, 2)
    holders[0] = 0b11
    got, mk = lib_plan(counts, holders, 2)
    assert 0 in got[0] and 0 in got[1]
    assert mk < 0.8 * mk0


@pytest.mark.parametrize("seed", range(20))
def test_one_replicated_expert_never_hurts(seed):
    # single-holder experts are placed first, so with one replicated expert
    # the plan can always fall back to its least-loaded holder
    rs = np.random.RandomState(100 + seed)
    world = int(rs.choice([2, 4, 8]))
    n_tok = int(rs.choice([512, 2048, 8192]))
    counts = rs.multinomial(2 * n_tok, rs.dirichlet(np.full(8, 0.5))).astype(np.int32)
    owner = np.arange(8) % world
    plain = (1 << owner).astype(np.uint32)
    rep = plain.copy()
    rep[int(np.argmax(counts))] = (1 << world) - 1
    _, mk0 = lib_plan(counts, plain, world)
    got, mk = lib_plan(counts, rep, world)
    assert mk <= mk0
    check_cover(got, counts, rep, world)


def test_measured_case_2048_tokens():
    # the routing tools/replica_proxy.py measured (hot expert 0, 2 ranks)
    counts = np.array([2048, 31, 22, 849, 110, 254, 12, 770], np.int32)
    owner = np.array([0, 1, 0, 1, 0, 1, 0, 1])
    plain = (1 << owner).astype(np.uint32)
    rep = plain.copy()
    rep[0] = 0b11
    _, mk0 = lib_plan(counts, plain, 2)
    got, mk = lib_plan(counts, rep, 2)
    assert mk < mk0
    assert 0 in got[0] and 0 in got[1]  # uneven split: most chunks on the light rank


def test_bad_arguments():
    with pytest.raises(M.MoeError):
        M.replica_plan([1, 2], [1, 1], 9, W_PS, ROW_PS, 0, CHUNK, 0)   # world > 8
    with pytest.raises(M.MoeError):
        M.replica_plan([1, 2], [1, 1], 2, W_PS, ROW_PS, 0, CHUNK, 2)   # rank >= world
    with pytest.raises(M.MoeError):
        M.replica_plan([1, -2], [1, 1], 2, W_PS, ROW_PS, 0, CHUNK, 0)  # negative count
