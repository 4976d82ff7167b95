"""Co-selection-aware expert-parallel shard map (moe_ep_shard_map_coselect,
shard_plan.h) on the host: against a brute-force restatement of its
objective, its balance constraint and its determinism; never worse than the
popularity LPT map (bench.shard_map / b200::ep_shard_map) on the objective.

The objective at batch 1 (top-2): a token whose two experts share a rank
streams both there, so the expected per-layer expert-streams are
1 + P(same rank); the map minimises the co-located co-selection count
(ties: the largest per-rank popularity load)."""
import itertools

import numpy as np
import pytest

import paper_2402_07033_b200 as M


def _cost(pairs, pop, owner, world):
    E = len(owner)
    c = sum(int(pairs[a, b] + pairs[b, a]) for a in range(E) for b in range(a + 1, E) if owner[a] == owner[b])
    load = max(sum(int(pop[e]) for e in range(E) if owner[e] == r) for r in range(world))
    return c, load


def _brute(pairs, pop, world):
    """Minimum (co-located co-selections, max load) over every balanced map."""
    E = len(pop)
    hi = -(-E // world)
    sizes_ok = (lambda sz: all(s == hi for s in sz)) if E % world == 0 else \
        (lambda sz: all(s in (hi - 1, hi) for s in sz) and sum(s == hi for s in sz) == E % world)
    best = None
    for owner in itertools.product(range(world), repeat=E):
        sz = [owner.count(r) for r in range(world)]
        if not sizes_ok(sz):
            continue
        c = _cost(pairs, pop, owner, world)
        best = c if best is None or c < best else best
    return best


def _lpt(pop, world):
    E = len(pop)
    owner = [0] * E
    cap = -(-E // world)
    load, held = [0] * world, [0] * world
    for e in sorted(range(E), key=lambda e: (-pop[e], e)):
        r = min((r for r in range(world) if held[r] < cap), key=lambda r: (load[r], r))
        owner[e] = r
        load[r] += pop[e]
        held[r] += 1
    return owner


def _random_layer(rs, E, skew):
    ids = []
    w = np.exp(skew * rs.randn(E))
    w /= w.sum()
    # correlated co-selection: a few favoured pairs
    fav = [tuple(rs.choice(E, 2, replace=False)) for _ in range(3)]
    for _ in range(400):
        if rs.rand() < 0.4:
            ids.append(fav[rs.randint(3)])
        else:
            ids.append(tuple(rs.choice(E, 2, replace=False, p=w)))
    pairs = np.zeros((E, E), np.int64)
    pop = np.zeros(E, np.int64)
    for a, b in ids:
        pairs[min(a, b), max(a, b)] += 1
        pop[a] += 1
        pop[b] += 1
    return pairs, pop


@pytest.mark.parametrize("E,world", [(8, 2), (8, 4), (6, 3), (7, 2), (8, 3), (5, 2), (4, 4), (8, 1)])
def test_coselect_map_is_optimal_and_balanced(E, world):
    rs = np.random.RandomState(E * 10 + world)
    L = 4
    pairs = np.zeros((L, E, E), np.int64)
    pop = np.zeros((L, E), np.int64)
    for l in range(L):
        pairs[l], pop[l] = _random_layer(rs, E, skew=0.7)
    owner, exact = M.ep_shard_map_coselect(pop, pairs, world)
    assert owner.shape == (L, E) and exact.all()
    for l in range(L):
        o = owner[l].tolist()
        assert all(0 <= r < world for r in o)
        sz = sorted(o.count(r) for r in range(world))
        assert sz[-1] - sz[0] <= 1, sz  # memory balance
        got = _cost(pairs[l], pop[l], o, world)
        assert got == _brute(pairs[l], pop[l], world), (l, o)
        assert got[0] <= _cost(pairs[l], pop[l], _lpt(pop[l].tolist(), world), world)[0]
    again, _ = M.ep_shard_map_coselect(pop, pairs, world)
    assert np.array_equal(owner, again)  # deterministic


def test_coselect_separates_a_dominant_pair():
    """Experts 0 and 2 are almost always chosen together: the LPT map of
    equal popularity puts them on one rank (0, 2, 4, 6 on rank 0); the
    co-selection map never does."""
    E, world = 8, 2
    pairs = np.zeros((1, E, E), np.int64)
    pairs[0, 0, 2] = 1000
    for a in range(E):
        for b in range(a + 1, E):
            pairs[0, a, b] += 1
    pop = np.full((1, E), 100, np.int64)
    lpt = _lpt(pop[0].tolist(), world)
    assert lpt[0] == lpt[2]
    owner, _ = M.ep_shard_map_coselect(pop, pairs, world)
    assert owner[0, 0] != owner[0, 2]


def test_coselect_large_E_local_search_and_errors():
    """E = 32 over 4 ranks exceeds the exact search's budget: the local
    search result is balanced and no worse than the LPT map; bad inputs are
    rejected."""
    E, world = 32, 4
    rs = np.random.RandomState(3)
    pairs, pop = _random_layer(rs, E, skew=0.5)
    owner, exact = M.ep_shard_map_coselect(pop[None], pairs[None], world)
    o = owner[0].tolist()
    assert sorted(o.count(r) for r in range(world)) == [8, 8, 8, 8]
    assert _cost(pairs, pop, o, world)[0] <= _cost(pairs, pop, _lpt(pop.tolist(), world), world)[0]
    with pytest.raises(M.MoeError):
        M.ep_shard_map_coselect(-pop[None], pairs[None], world)
    with pytest.raises(M.MoeError):
        M.ep_shard_map_coselect(pop[None], pairs[None], 0)
