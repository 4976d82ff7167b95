"""Pins the C oracle (oracle/moe_oracle.c) to the reference.

Every assertion here is either a known answer from the reference's own tests
(proj/tests/test_model.cpp, test_placement.cpp, acceptance.cpp) or a golden
vector produced by the reference itself (tests/golden/make_golden.py).  fp64
values must match BIT-EXACTLY: the oracle restates the reference's operation
order and is compiled without FMA contraction.
"""
import math

import numpy as np
import pytest

import oracle as O


def _split(flat):
    """Decode the length-prefixed record arrays written by make_golden.py."""
    n = 0
    lens = []
    i = 0
    # header: first all lengths (one per record) until they sum to the tail
    while True:
        lens.append(int(flat[i]))
        i += 1
        if i + sum(lens) == len(flat):
            break
    out = []
    for ln in lens:
        out.append(flat[i:i + ln])
        i += ln
    return out


def test_known_answers_silu(orc):
    # test_model.cpp:65-70
    assert orc.silu(0.0) == 0.0
    assert abs(orc.silu(20.0) - 20.0) <= 1e-6 * 20.0
    assert abs(orc.silu(1.0) - 0.7310585786300049) <= 1e-12


def test_expert_ffn_zero_and_identity(orc):
    # test_model.cpp:72-90
    y = orc.expert_ffn(np.zeros((4, 3)), np.zeros((4, 3)), np.zeros((3, 4)), [1.0, -2.0, 0.5])
    assert (y == 0).all()
    one = np.ones((1, 1))
    assert abs(orc.expert_ffn(one, one, one, [1.0])[0] - 0.7310585786300049) <= 1e-12


def test_expert_ffn_instances_bitexact(orc, golden):
    # random instances in the shape ranges of test_model.cpp:92-107, answers
    # from the reference's expert_ffn.
    for rec in _split(golden["ffn_inst"]):
        d, f = int(rec[0]), int(rec[1])
        o = 2
        wi = rec[o:o + f * d].reshape(f, d); o += f * d
        wg = rec[o:o + f * d].reshape(f, d); o += f * d
        wo = rec[o:o + d * f].reshape(d, f); o += d * f
        x = rec[o:o + d]; o += d
        want = rec[o:o + d]
        assert np.array_equal(orc.expert_ffn(wi, wg, wo, x), want)


def test_gate_topk_known_answers(orc, golden):
    # test_model.cpp:132-159
    ids, w, _ = orc.gate_topk(np.array([[3.0], [1.0], [1.0], [1.0]]), [1.0], 2)
    assert list(ids) == [0, 1]
    assert abs(w[0] - 0.8807970779778823) <= 1e-12
    assert abs(w[1] - 0.11920292202211755) <= 1e-12
    ids, w, _ = orc.gate_topk(np.full((4, 1), 2.0), [1.0], 2)
    assert list(ids) == [0, 1] and w[0] == pytest.approx(0.5) and w[1] == pytest.approx(0.5)
    for rec in _split(golden["topk"]):
        E, k = int(rec[0]), int(rec[1])
        logits = rec[2:2 + E]
        ids, w, _ = orc.gate_topk(logits[:, None], [1.0], k)
        assert list(ids) == list(rec[2 + E:2 + E + k].astype(int))
        assert np.array_equal(w, rec[2 + E + k:2 + E + 2 * k])
        # test_model.cpp:161-180: positive, sum to 1, shift invariance
        assert (w > 0).all() and abs(w.sum() - 1.0) <= 1e-9
        ids2, _, _ = orc.gate_topk((logits + 5.0)[:, None], [1.0], k)
        assert list(ids2) == list(ids)


def test_gate_topk_rejects_bad_k(orc):
    with pytest.raises(ValueError):
        orc.gate_topk(np.ones((3, 1)), [1.0], 0)
    with pytest.raises(ValueError):
        orc.gate_topk(np.ones((3, 1)), [1.0], 4)


@pytest.mark.parametrize("name,seed", [("toy_s3", 3), ("crit8", 8), ("crit9", 9)])
def test_random_model_and_forward_bitexact(orc, golden, name, seed):
    toy = O.Shape(4, 8, 2, 32, 64, 2)
    w = orc.random_model(toy, seed)
    assert np.array_equal(w.w_in[0], golden[f"{name}_w_in0"])
    assert np.array_equal(w.router[3], golden[f"{name}_router3"])
    sums = np.array([sum(float(m.sum()) for m in w.w_in), sum(float(m.sum()) for m in w.w_gate),
                     sum(float(m.sum()) for m in w.w_out), sum(float(m.sum()) for m in w.router)])
    assert np.array_equal(sums, golden[f"{name}_wsum"])
    calls = []
    out, tally, gsum, ids, gates = orc.model_forward(toy, w, golden[f"{name}_tokens"],
                                                     sink=lambda l, v: calls.append(v))
    assert np.array_equal(out, golden[f"{name}_out"])
    assert np.array_equal(tally, golden[f"{name}_count"])
    mean_gate = np.where(tally > 0, gsum / np.maximum(tally, 1), 0.0)
    assert np.array_equal(mean_gate, golden[f"{name}_gate"])
    assert np.array_equal(np.concatenate(calls), golden[f"{name}_sink"])
    # trace invariants (trace.cpp:59-79): prefill totals = tokens*k per layer
    n = golden[f"{name}_tokens"].shape[0]
    assert (tally.sum(axis=1) == n * toy.top_k).all()


def test_sparsity_histogram(orc, golden):
    thr = [0.001, 0.01, 0.1, 1.0]
    assert list(orc.sparsity_histogram([0.0005, 0.05, 0.5, 2.0], thr)) == [0.25, 0.25, 0.5, 0.75]
    assert np.array_equal(orc.sparsity_histogram([0.0005, 0.05, 0.5, 2.0], thr),
                          golden["hand_hist"])
    sink = golden["crit9_sink"].reshape(16, 4, 2, 64)
    for l in range(4):
        h = orc.sparsity_histogram(sink[:, l].reshape(-1), thr)
        assert np.array_equal(h, golden["crit9_hist"][l])
        assert (np.diff(h) >= 0).all()  # acceptance.cpp criterion 9


def test_single_layer_hand_composed(orc, golden):
    s1 = O.Shape(1, 2, 2, 3, 4, 2)
    w = orc.random_model(s1, 42)
    flat = np.concatenate([w.w_in[0].ravel(), w.w_gate[0].ravel(), w.w_out[0].ravel(),
                           w.w_in[1].ravel(), w.w_gate[1].ravel(), w.w_out[1].ravel(),
                           w.router[0].ravel()])
    assert np.array_equal(flat, golden["s42_w"])
    out, tally, gsum, _, _ = orc.model_forward(s1, w, np.array([[0.3, -0.7, 1.1]]))
    assert np.array_equal(out, golden["s42_out"])


def test_tiny_config_probe_values(orc, golden):
    # SURVEY §8c probe (T): weights, selection and outputs from the reference.
    T = O.Shape(1, 8, 2, 512, 1792, 4)
    w = orc.random_model(T, 0)
    assert w.w_in[0][0, 0] == 0.0045042063583167098
    assert w.router[0][0, 1] == 0.019798144683463425
    assert np.array_equal(w.router[0], golden["T_router"])
    for e in range(8):
        assert np.array_equal(w.w_in[e][0, :4], golden["T_samples"][e, 0])
        assert np.array_equal(w.w_out[e][7, :4], golden["T_samples"][e, 2])
        assert float(w.w_gate[e].sum()) == golden["T_wsum"][e, 1]
    x = orc.normal(1, 512)[None]
    assert np.array_equal(x, golden["T_token"])
    out, tally, gsum, ids, gates = orc.model_forward(T, w, x)
    assert list(ids[0, 0]) == [1, 4]
    assert np.array_equal(out, golden["T_out"])
    # SURVEY's probe (different build flags) agrees to ~1 ulp
    assert abs(out[0, 0] - -0.89580440859426269) < 1e-14


def test_mixtral_layer_probe(golden):
    # Recorded from the reference at d=4096,f=14336: selection
    # (e1, 0.36698151487136049), (e2, 0.63301848512863956).
    if "M_count" not in golden.files:
        pytest.skip("golden generated without --mixtral")
    assert list(np.nonzero(golden["M_count"][0])[0]) == [1, 2]
    assert golden["M_gate"][0, 1] == 0.36698151487136049
    assert abs(golden["M_out"][0, 0] - -0.45676723825482834) < 1e-14


def test_placement_against_reference_goldens(orc, golden):
    # greedy_place / expected_hit_rate / hit_rate_bounds (placement.cpp:68-124)
    for rec in _split(golden["placement"]):
        L, E, cap = int(rec[0]), int(rec[1]), int(rec[2])
        o = 3
        counts = rec[o:o + L * E].reshape(L, E).astype(np.int64); o += L * E
        res = rec[o:o + L * E].reshape(L, E); o += L * E
        resq = rec[o:o + L * E].reshape(L, E); o += L * E
        hr = rec[o]; b = rec[o + 1:o + 4]
        total = int(counts.sum())
        assert np.array_equal(orc.greedy_place(counts, cap), res)
        assert np.array_equal(orc.greedy_place(counts, cap, per_layer_quota=True), resq)
        assert orc.expected_hit_rate(res, counts, total) == hr
        assert np.array_equal(np.array(orc.hit_rate_bounds(counts, total, cap)), b)


def test_placement_known_answers(orc):
    # test_placement.cpp:103-147
    strict = np.array([[12, 7, 3], [9, 5, 1]])
    assert set(zip(*np.nonzero(orc.greedy_place(strict, 3)))) == {(0, 0), (1, 0), (0, 1)}
    tie = np.array([[5, 5], [5, 5]])
    assert set(zip(*np.nonzero(orc.greedy_place(tie, 3)))) == {(0, 0), (0, 1), (1, 0)}
    p = np.array([[9, 8, 1], [2, 1, 0]])
    assert set(zip(*np.nonzero(orc.greedy_place(p, 2)))) == {(0, 0), (0, 1)}
    assert set(zip(*np.nonzero(orc.greedy_place(p, 2, True)))) == {(0, 0), (1, 0)}
    u = np.ones((32, 8), np.int64)
    assert orc.expected_hit_rate(orc.greedy_place(u, 56), u, 256) == 0.21875
    assert orc.expected_hit_rate(orc.greedy_place(u, 52), u, 256) == 0.203125
    with pytest.raises(ValueError):
        orc.expected_hit_rate(np.zeros((1, 2), np.uint8), np.zeros((1, 2)), 0)
    b = orc.hit_rate_bounds(np.array([[3, 1]]), 4, 1)
    assert b == (0.75, 0.25, 0.5)


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random_shapes(orc):
    """Cross-check against the reference library itself on random small shapes."""
    ref = O.Reference()
    rs = np.random.RandomState(3)
    for trial in range(12):
        s = O.Shape(int(rs.randint(0, 4)), int(rs.randint(2, 9)), 1, int(rs.randint(1, 24)),
                    int(rs.randint(1, 40)), 2)
        s = O.Shape(s.num_layers, s.experts_per_layer, int(rs.randint(1, s.experts_per_layer + 1)),
                    s.hidden_dim, s.ffn_dim, 2)
        seed = int(rs.randint(1 << 30))
        wo, wr = orc.random_model(s, seed), ref.random_model(s, seed)
        for a, b in zip(wo.w_in + wo.w_out + wo.router, wr.w_in + wr.w_out + wr.router):
            assert np.array_equal(a, b)
        toks = rs.randn(int(rs.randint(1, 5)), s.hidden_dim)
        out_o = orc.model_forward(s, wo, toks)
        out_r = ref.model_forward(s, wr, toks)
        assert np.array_equal(out_o[0], out_r[0])
        assert np.array_equal(out_o[1], out_r[1])


def test_random_model_stream_equals_random_model(orc):
    """The streamed random_model (one expert at a time, used to upload the
    reference's Mixtral layer to the GPU) draws exactly random_model's values."""
    sh = O.Shape(2, 4, 2, 16, 24, 2)
    w = orc.random_model(sh, 5)
    n = 0
    for it in orc.random_model_stream(sh, 5):
        if it[0] == "expert":
            _, l, e, a, b, c = it
            wa, wb, wc = w.expert(l, e)
            assert np.array_equal(a, wa) and np.array_equal(b, wb) and np.array_equal(c, wc)
        else:
            _, l, r = it
            assert np.array_equal(r, w.router[l])
        n += 1
    assert n == 2 * 4 + 2


def test_expert_ffn_batch_is_bitwise_expert_ffn(orc):
    rs = np.random.RandomState(1)
    for d, f, n in [(3, 5, 1), (16, 24, 7), (64, 32, 3)]:
        wi, wg, wo = rs.randn(f, d), rs.randn(f, d), rs.randn(d, f)
        X = rs.randn(n, d)
        Y = orc.expert_ffn_batch(wi, wg, wo, X)
        for t in range(n):
            assert np.array_equal(Y[t], orc.expert_ffn(wi, wg, wo, X[t]))
