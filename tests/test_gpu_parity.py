"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Protocol: the oracle is fed the values the device actually holds
(weights downloaded after RNE rounding, tokens rounded to fp32), so the
tolerance measures kernel arithmetic, not quantisation.
  * routing ids / counts / permutation: bit-exact (near-ties, margin below
    1e-5*max|logit|, are reported and excluded — none occur at these seeds);
  * outputs: normwise max|gpu-ref| / max|ref| on the MoE delta (out - x):
    <= 1e-5 in fp32 mode, <= 1e-2 in bf16 mode (north_star).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_2402_07033_b200 as M  # noqa: E402

TOL_F32 = 1e-5
TOL_BF16 = 1e-2


def normwise(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()
    c = M.Ctx(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def orc():
    O.build(ref=False)
    return O.Oracle()


def margin(logits, k):
    s = np.sort(logits)[::-1]
    return (s[k - 1] - s[k]) / max(np.abs(logits).max(), 1e-30) if k < len(s) else np.inf


def oracle_layer(orc, w, l, x, k):
    """Oracle layer on device-held values: returns (ids, gates, delta, margin)."""
    router = w.download_router(l)
    ids, g, logits = orc.gate_topk(router, x, k)
    delta = np.zeros_like(x)
    for e, ge in zip(ids, g):
        wi, wg, wo = w.download_expert(l, int(e))
        delta += ge * orc.expert_ffn(wi, wg, wo, x)
    return ids, g, delta, margin(logits, k)


# ---------------------------------------------------------------------------
def test_library_reports_streaming_decode(ctx):
    s = M.Shape(1, 8, 2, 4096, 14336, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    assert w.expert_path(1) == 1          # TMA-ring streaming kernel
    assert w.expert_path(4) == 3            # tcgen05 grouped GEMM (prefill)
    assert w.forward_launches(1) == 1       # persistent stack kernel
    w.close()


def test_router_topk_bitexact_ids(ctx, orc):
    s = M.Shape(1, 8, 2, 512, 1792, 4)
    w = M.Weights(ctx, s, M.DTYPE_F32)
    ow = orc.random_model(O.Shape(1, 8, 2, 512, 1792, 4), 0)
    w.upload_router(0, ow.router[0])
    router = w.download_router(0)
    rs = np.random.RandomState(0)
    n = 256
    x = f32(rs.randn(n, 512))
    xd = torch.tensor(x, dtype=torch.float32, device="cuda")
    ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
    gates = torch.zeros((n, 2), dtype=torch.float32, device="cuda")
    w.router_topk(0, xd, ids, gates)
    torch.cuda.synchronize()
    ids, gates = ids.cpu().numpy(), gates.cpu().numpy()
    near = 0
    for t in range(n):
        want_ids, want_g, logits = orc.gate_topk(router, x[t], 2)
        if margin(logits, 2) < 1e-5:
            near += 1
            continue
        assert list(ids[t]) == list(want_ids)
        assert np.abs(gates[t] - want_g).max() < 1e-5
    assert near == 0


def test_router_tie_break_known_answers(ctx):
    # test_model.cpp:132-159 through the device router
    ids, g = ctx.gate_topk_host(np.array([[3.0], [1.0], [1.0], [1.0]]), np.array([1.0]), 2)
    assert list(ids) == [0, 1]
    assert abs(g[0] - 0.8807970779778823) < 1e-6 and abs(g[1] - 0.11920292202211755) < 1e-6
    ids, g = ctx.gate_topk_host(np.full((4, 1), 2.0), np.array([1.0]), 2)
    assert list(ids) == [0, 1] and abs(g[0] - 0.5) < 1e-7
    ids, g = ctx.gate_topk_host(np.array([[1.0], [2.0], [3.0]]), np.array([1.0]), 3)
    den = np.exp([1.0, 2.0, 3.0]).sum()
    assert np.allclose(g, np.exp([1.0, 2.0, 3.0]) / den, atol=1e-6)
    with pytest.raises(M.MoeError) as ei:
        ctx.gate_topk_host(np.ones((3, 1)), np.array([1.0]), 4)
    assert ei.value.kind == "ShapeError"


def test_expert_ffn_small_shapes(ctx, orc):
    # the shape range of test_model.cpp:92-107, fp32 mode
    rs = np.random.RandomState(7)
    for _ in range(40):
        d, f = 2 + rs.randint(5), 2 + rs.randint(7)
        wi, wg, wo, x = f32(rs.randn(f, d)), f32(rs.randn(f, d)), f32(rs.randn(d, f)), f32(rs.randn(d))
        got = ctx.expert_ffn_host(M.DTYPE_F32, wi, wg, wo, x)
        assert normwise(got, orc.expert_ffn(wi, wg, wo, x)) < TOL_F32
    one = np.ones((1, 1))
    assert abs(ctx.expert_ffn_host(M.DTYPE_F32, one, one, one, np.ones(1))[0] - 0.7310585786300049) < 1e-6
    z = ctx.expert_ffn_host(M.DTYPE_F32, np.zeros((4, 3)), np.zeros((4, 3)), np.zeros((3, 4)),
                            np.array([1.0, -2.0, 0.5]))
    assert (z == 0).all()


@pytest.mark.parametrize("name,seed", [("toy_s3", 3), ("crit8", 8)])
def test_forward_host_toy_vs_reference_golden(ctx, orc, golden, name, seed):
    """Full model_forward on the toy shape (4 layers, d=32): GPU vs the
    reference's own outputs (tests/golden), fp32 mode."""
    toy = O.Shape(4, 8, 2, 32, 64, 2)
    ow = orc.random_model(toy, seed)
    w = M.Weights(ctx, M.Shape(4, 8, 2, 32, 64, 2), M.DTYPE_F32)
    w.upload_oracle(ow)
    toks = golden[f"{name}_tokens"]
    out, ids, gates = w.forward_host(toks)
    want = golden[f"{name}_out"]
    assert normwise(out - toks, want - toks) < 1e-4  # fp32 weights+tokens vs fp64 reference
    counts = np.zeros((4, 8), np.int64)
    for l in range(4):
        for e in ids[l].ravel():
            counts[l, e] += 1
    assert np.array_equal(counts, golden[f"{name}_count"])
    # determinism (test_model.cpp:217-231 / criterion 8): bit-identical reruns
    out2, ids2, gates2 = w.forward_host(toks)
    assert np.array_equal(out, out2) and np.array_equal(ids, ids2) and np.array_equal(gates, gates2)


def test_sink_post_silu_matches_reference(ctx, orc, golden):
    """ActivationSink values (model.cpp:131-139) in reference call order."""
    toy = O.Shape(4, 8, 2, 32, 64, 2)
    ow = orc.random_model(toy, 9)
    w = M.Weights(ctx, M.Shape(4, 8, 2, 32, 64, 2), M.DTYPE_F32)
    w.upload_oracle(ow)
    toks = golden["crit9_tokens"]
    out, ids, gates, post = w.forward_host(toks, with_post=True)
    want = golden["crit9_sink"]
    assert post.shape == want.shape
    assert normwise(post, want) < 1e-4
    thr = [0.001, 0.01, 0.1, 1.0]
    sink = post.reshape(16, 4, 2, 64)
    for l in range(4):
        h = orc.sparsity_histogram(sink[:, l].reshape(-1), thr)
        assert (np.diff(h) >= 0).all()


def test_tiny_layer_decode_fp32(ctx, orc, golden):
    """Config T (d=512, f=1792, fp32, batch 1) on the streaming decode kernel,
    against the reference's golden output."""
    T = O.Shape(1, 8, 2, 512, 1792, 4)
    ow = orc.random_model(T, 0)
    w = M.Weights(ctx, M.Shape(1, 8, 2, 512, 1792, 4), M.DTYPE_F32)
    assert w.expert_path(1) == 1
    w.upload_oracle(ow)
    x = golden["T_token"]
    out, ids, gates = w.forward_host(x)
    assert list(ids[0, 0]) == [1, 4]
    assert normwise(out - x, golden["T_out"] - x) < TOL_F32 * 10
    # strict protocol: oracle on the fp32-rounded token
    xr = f32(x[0])
    _, _, delta, _ = oracle_layer(orc, w, 0, xr, 2)
    xd = torch.tensor(xr[None], dtype=torch.float32, device="cuda")
    idd = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    gd = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    xo = torch.empty_like(xd)
    w.layer_forward(0, xd, xo, idd, gd)
    torch.cuda.synchronize()
    assert normwise(xo.cpu().numpy()[0].astype(np.float64) - xr, delta) < TOL_F32


def test_mixtral_layer_decode_bf16(ctx, orc, golden):
    """Config M: Mixtral-8x7B-shaped layer, bf16 weights (device Philox init),
    batch-1 decode through the TMA-ring kernel."""
    s = M.Shape(1, 8, 2, 4096, 14336, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    w.random(0)
    x = f32(golden["M_token"][0])
    xd = torch.tensor(x[None], dtype=torch.float32, device="cuda")
    idd = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    gd = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    xo = torch.empty_like(xd)
    w.layer_forward(0, xd, xo, idd, gd)
    torch.cuda.synchronize()
    ids, g, delta, mg = oracle_layer(orc, w, 0, x, 2)
    assert mg > 1e-5
    assert list(idd.cpu().numpy()[0]) == list(ids)
    assert np.abs(gd.cpu().numpy()[0] - g).max() < 1e-5
    err = normwise(xo.cpu().numpy()[0].astype(np.float64) - x, delta)
    print(f"M bf16 normwise error {err:.3e}")
    assert err < TOL_BF16
    assert err < 1e-4  # fp32 accumulation of exactly-represented bf16 weights


def test_mixtral_layer_decode_fp32_mode(ctx, orc, golden):
    s = M.Shape(1, 8, 2, 4096, 14336, 4)
    w = M.Weights(ctx, s, M.DTYPE_F32)
    assert w.expert_path(1) == 1
    w.random(1)
    x = f32(golden["M_token"][0])
    xd = torch.tensor(x[None], dtype=torch.float32, device="cuda")
    idd = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    gd = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    xo = torch.empty_like(xd)
    w.layer_forward(0, xd, xo, idd, gd)
    torch.cuda.synchronize()
    ids, g, delta, mg = oracle_layer(orc, w, 0, x, 2)
    assert list(idd.cpu().numpy()[0]) == list(ids)
    assert normwise(xo.cpu().numpy()[0].astype(np.float64) - x, delta) < TOL_F32


def test_stack_decode_teacher_forced_and_graph(ctx, orc):
    """4-layer Mixtral-shaped stack: per-layer teacher-forced parity, then the
    single-graph moe_forward must agree with the layer-by-layer chain and be
    bit-deterministic across runs."""
    L = 4
    s = M.Shape(L, 8, 2, 4096, 14336, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    w.random(7)
    x0 = f32(orc.normal(1, 4096))
    xs = [torch.tensor(x0[None], dtype=torch.float32, device="cuda")]
    ids_l = []
    for l in range(L):
        xo = torch.empty_like(xs[-1])
        idd = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
        gd = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
        w.layer_forward(l, xs[-1], xo, idd, gd)
        torch.cuda.synchronize()
        xin = xs[-1].cpu().numpy()[0].astype(np.float64)
        ids, g, delta, mg = oracle_layer(orc, w, l, xin, 2)
        assert list(idd.cpu().numpy()[0]) == list(ids), f"layer {l}"
        assert normwise(xo.cpu().numpy()[0].astype(np.float64) - xin, delta) < TOL_BF16
        ids_l.append(list(ids))
        xs.append(xo)
    # fused graph path
    xg = torch.tensor(x0[None], dtype=torch.float32, device="cuda")
    idg = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    gg = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
    w.forward(xg, idg, gg)
    torch.cuda.synchronize()
    assert [list(r) for r in idg.cpu().numpy()[:, 0]] == ids_l
    ref = xs[-1].cpu().numpy()[0].astype(np.float64)
    assert normwise(xg.cpu().numpy()[0] - x0, ref - x0) < 1e-4
    out1 = xg.clone()
    for _ in range(3):
        xg.copy_(torch.tensor(x0[None], dtype=torch.float32, device="cuda"))
        w.forward(xg, idg, gg)
        torch.cuda.synchronize()
        assert torch.equal(xg, out1)


def test_prefill_generic_tokens_T(ctx, orc):
    """Multi-token forward (prefill step) on config T, fp32: outputs and the
    per-(layer,expert) tally (the RoutingTrace) against the oracle."""
    T = O.Shape(2, 8, 2, 512, 1792, 4)
    ow = orc.random_model(T, 5)
    w = M.Weights(ctx, M.Shape(2, 8, 2, 512, 1792, 4), M.DTYPE_F32)
    w.upload_oracle(ow)
    toks = f32(orc.normal(6, 16 * 512).reshape(16, 512))
    out, ids, gates = w.forward_host(toks)
    # oracle on device-rounded weights
    dw = O.Weights(T)
    for e in range(8):
        for l in range(2):
            a, b, c = w.download_expert(l, e)
            i = l * 8 + e
            dw.w_in[i][:], dw.w_gate[i][:], dw.w_out[i][:] = a, b, c
    for l in range(2):
        dw.router[l][:] = w.download_router(l)
    want, tally, gsum, want_ids, want_g = orc.model_forward(T, dw, toks)
    assert np.array_equal(ids.transpose(1, 0, 2), want_ids)
    assert normwise(out - toks, want - toks) < TOL_F32 * 10


def test_permute_stable_and_deterministic(ctx):
    rs = np.random.RandomState(3)
    for n_tok, k, E in [(1, 2, 8), (512, 2, 8), (1000, 3, 16), (4097, 2, 64)]:
        ids = np.stack([np.sort(rs.choice(E, k, replace=False)) for _ in range(n_tok)]).astype(np.int32)
        d_ids = torch.tensor(ids, device="cuda")
        counts = torch.zeros(E, dtype=torch.int32, device="cuda")
        offsets = torch.zeros(E, dtype=torch.int32, device="cuda")
        perm = torch.zeros(n_tok * k, dtype=torch.int32, device="cuda")
        inv = torch.zeros(n_tok * k, dtype=torch.int32, device="cuda")
        ctx.permute(d_ids, n_tok, k, E, counts, offsets, perm, inv)
        torch.cuda.synchronize()
        flat = ids.ravel()
        want_perm = np.argsort(flat, kind="stable")
        assert np.array_equal(perm.cpu().numpy(), want_perm)
        assert np.array_equal(counts.cpu().numpy(), np.bincount(flat, minlength=E))
        assert np.array_equal(inv.cpu().numpy()[want_perm], np.arange(n_tok * k))


def test_errors_are_loud(ctx):
    s = M.Shape(2, 4, 2, 16, 32, 2)
    w = M.Weights(ctx, s, M.DTYPE_F32)
    with pytest.raises(M.MoeError) as ei:
        w.download_router(5)
    assert ei.value.kind == "ShapeError"
    with pytest.raises(M.MoeError) as ei:
        M.Weights(ctx, M.Shape(1, 2, 3, 16, 32, 2))
    assert ei.value.kind == "ShapeError"


@pytest.mark.parametrize("L,d,f,dt", [(4, 4096, 14336, M.DTYPE_BF16), (3, 512, 1792, M.DTYPE_F32),
                                      (2, 6144, 16384, M.DTYPE_BF16)])
def test_persistent_stack_matches_per_layer_path(ctx, orc, L, d, f, dt, libopts):
    """The one-launch persistent stack kernel against the per-layer 2-kernel
    path on identical weights: same routing, outputs within fp32 rounding."""
    s = M.Shape(L, 8, 2, d, f, 2 if dt == M.DTYPE_BF16 else 4)
    w_stack = M.Weights(ctx, s, dt)
    libopts(stack=0)
    w_layer = M.Weights(ctx, s, dt)
    libopts(stack=1)
    assert w_stack.forward_launches(1) == 1 and w_layer.forward_launches(1) == 1 + 2 * L
    w_stack.random(11)
    w_layer.random(11)
    x0 = f32(orc.normal(2, d))
    outs, idss = [], []
    for w in (w_stack, w_layer):
        x = torch.tensor(x0[None], dtype=torch.float32, device="cuda")
        ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
        w.forward(x, ids, g)
        torch.cuda.synchronize()
        outs.append(x.cpu().numpy()[0].astype(np.float64))
        idss.append(ids.cpu().numpy())
    assert np.array_equal(idss[0], idss[1])
    assert normwise(outs[0] - x0, outs[1] - x0) < 1e-4
    # teacher-forced oracle check of the stack's first layer
    ids, gts, delta, mg = oracle_layer(orc, w_stack, 0, x0, 2)
    assert list(idss[0][0, 0]) == list(ids)
    w_stack.close()
    w_layer.close()


def _prefill_case(ctx, orc, libopts, L, d, f, n_tok, seed, sample):
    s = M.Shape(L, 8, 2, d, f, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    assert w.expert_path(n_tok) == 3  # tcgen05 grouped GEMM
    libopts(prefill=0)
    wg = M.Weights(ctx, s, M.DTYPE_BF16)
    libopts(prefill=1)
    assert wg.expert_path(n_tok) == 2
    w.random(seed)
    wg.random(seed)
    rs = np.random.RandomState(seed)
    x = f32(rs.randn(n_tok, d))
    outs = []
    for ww in (w, wg):
        xd = torch.tensor(x, dtype=torch.float32, device="cuda")
        xo = torch.empty_like(xd)
        ids = torch.zeros((n_tok, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((n_tok, 2), dtype=torch.float32, device="cuda")
        ww.layer_forward(0, xd, xo, ids, g)
        torch.cuda.synchronize()
        outs.append((xo.cpu().numpy().astype(np.float64), ids.cpu().numpy(), g.cpu().numpy()))
    (o_tc, id_tc, g_tc), (o_gen, id_gen, g_gen) = outs
    assert np.array_equal(id_tc, id_gen)
    err_gen = normwise(o_tc - x, o_gen - x)
    print(f"prefill tcgen05 vs generic CUDA: {err_gen:.3e}")
    assert err_gen < TOL_BF16
    # oracle on device-held weights for a sample of tokens
    router = w.download_router(0)
    cache = {}
    worst = 0.0
    for t in sample:
        ids, gts, logits = orc.gate_topk(router, x[t], 2)
        assert list(id_tc[t]) == list(ids)
        delta = np.zeros(d)
        for e, ge in zip(ids, gts):
            if e not in cache:
                cache[e] = w.download_expert(0, int(e))
            delta += ge * orc.expert_ffn(*cache[e], x[t])
        worst = max(worst, normwise(o_tc[t] - x[t], delta))
    print(f"prefill tcgen05 vs oracle (sample of {len(sample)}): {worst:.3e}")
    assert worst < TOL_BF16
    w.close()
    wg.close()


def test_prefill_tcgen05_small_uneven(ctx, orc, libopts):
    """d=256, f=512, 700 tokens: experts see >256 tokens (2 N-chunks), ragged
    tails, every token checked against the oracle."""
    _prefill_case(ctx, orc, libopts, 1, 256, 512, 700, 3, range(0, 700, 7))


def test_prefill_tcgen05_mixtral_layer_512(ctx, orc, libopts):
    """Config P: Mixtral-shaped layer, 512-token prefill on the tcgen05 path."""
    _prefill_case(ctx, orc, libopts, 1, 4096, 14336, 512, 5, [0, 1, 77, 200, 311, 511])


@pytest.mark.parametrize("late8,cut16", [(8, 14), (3, 12)])
def test_prefill_uneven_k_split(ctx, orc, libopts, late8, cut16):
    """Down tiles split 2-way at cut16/16 of K with the small pieces
    scheduled last (pf_cut16): still within tolerance of the generic CUDA
    path and the oracle, at the Mixtral shape and the ragged small one."""
    libopts(pf_late8=late8, pf_cut16=cut16)
    _prefill_case(ctx, orc, libopts, 1, 4096, 14336, 512, 5, [0, 1, 77, 200, 311, 511])
    _prefill_case(ctx, orc, libopts, 1, 256, 512, 700, 3, range(0, 700, 7))


@pytest.mark.parametrize("n_tok", [512, 700])
def test_combine_k2_equals_looped_combine(ctx, libopts, n_tok):
    """The top-2 combine that issues all loads up front (combine_k2_kernel)
    is bit-identical to the looped combine (debug option combine4) on the
    tcgen05 prefill path, K-split partials included."""
    w = M.Weights(ctx, M.Shape(1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
    w.random(3)
    x = torch.randn(n_tok, 4096, device="cuda")
    outs = []
    for env in (0, 1):
        libopts(combine4=env)
        o = torch.empty_like(x)
        ids = torch.zeros((n_tok, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((n_tok, 2), device="cuda")
        w.layer_forward(0, x, o, ids, g)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
    w.close()


@pytest.mark.parametrize("n_tok", [1, 300, 512])
def test_forward_host_equals_device_path(ctx, n_tok):
    """The fp64 host-buffer entry point (pooled conversion, chunked copies for
    prefill sizes) gives exactly moe_forward's result on the same fp32 tokens
    (batch 1: the same captured stack-kernel graph): out == double(device
    out), ids and gates equal."""
    w = M.Weights(ctx, M.Shape(1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
    w.random(4)
    xh = np.random.RandomState(n_tok).randn(n_tok, 4096)
    out, ids_h, g_h = w.forward_host(xh)
    o = torch.tensor(xh.astype(np.float32), device="cuda")  # moe_forward: in place
    ids = torch.zeros((1, n_tok, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((1, n_tok, 2), device="cuda")
    w.forward(o, ids, g)
    torch.cuda.synchronize()
    assert np.array_equal(out, o.cpu().numpy().astype(np.float64))
    assert np.array_equal(ids_h, ids.cpu().numpy())
    assert np.array_equal(g_h, g.cpu().numpy().astype(np.float64))
    w.close()


def test_kernel_timing_counts_grouped_launches(ctx):
    """moe_debug_kernel_timing: one event pair per tcgen05 grouped launch,
    none for batch-1 calls; results unchanged while timing."""
    w = M.Weights(ctx, M.Shape(1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
    w.random(2)
    x = torch.randn(512, 4096, device="cuda")
    o0, o1 = torch.empty_like(x), torch.empty_like(x)
    ids = torch.zeros((512, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((512, 2), device="cuda")
    w.layer_forward(0, x, o0, ids, g)
    w.kernel_timing(True)
    for _ in range(3):
        w.layer_forward(0, x, o1, ids, g)
    w.layer_forward(0, x[:1], o1[:1], ids[:1], g[:1])  # decode path: not timed
    tot, n = w.kernel_timing(False)
    torch.cuda.synchronize()
    assert n == 3 and 100.0 < tot / n < 5000.0
    w.layer_forward(0, x, o1, ids, g)
    torch.cuda.synchronize()
    assert torch.equal(o0, o1)
    w.close()


def test_router_many_tokens_batched_kernel(ctx, orc):
    """The router's per-token arithmetic does not depend on n_tok or on the
    token's slot in a block: one 4100-token call equals 1000-token chunks bit
    for bit, and ids match the fp64 oracle away from near-ties."""
    s = M.Shape(1, 8, 2, 512, 1792, 4)
    w = M.Weights(ctx, s, M.DTYPE_F32)
    ow = orc.random_model(O.Shape(1, 8, 2, 512, 1792, 4), 1)
    w.upload_router(0, ow.router[0])
    n = 4100
    x = torch.randn(n, 512, device="cuda")
    ids = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((n, 2), dtype=torch.float32, device="cuda")
    w.router_topk(0, x, ids, g)
    ids1 = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
    g1 = torch.zeros((n, 2), dtype=torch.float32, device="cuda")
    for c0 in range(0, n, 1001):  # chunks that shift the block alignment
        c1 = min(n, c0 + 1001)
        w.router_topk(0, x[c0:c1], ids1[c0:c1], g1[c0:c1])
    torch.cuda.synchronize()
    assert torch.equal(ids, ids1) and torch.equal(g, g1)
    router = w.download_router(0)
    xs = x.cpu().numpy().astype(np.float64)
    for t in range(0, n, 97):
        want, _, logits = orc.gate_topk(router, xs[t], 2)
        if margin(logits, 2) > 1e-5:
            assert list(ids[t].cpu().numpy()) == list(want)


def test_routing_histogram_and_shard_map(ctx):
    """Device routing histogram (f1): counts over a multi-layer forward's ids
    equal a host bincount, accumulate across calls, and feed the shard map."""
    import importlib.util
    import os
    L, E, k, d, f, n = 3, 8, 2, 512, 1792, 200
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 4), M.DTYPE_F32)
    w.random(5)
    x = torch.randn(n, d, device="cuda")
    ids = torch.zeros((L, n, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, n, k), device="cuda")
    w.forward(x, ids, g)
    counts = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    ctx.routing_histogram(ids, counts)
    ctx.routing_histogram(ids, counts)
    torch.cuda.synchronize()
    host = ids.cpu().numpy()
    want = np.stack([np.bincount(host[l].ravel(), minlength=E) for l in range(L)])
    assert np.array_equal(counts.cpu().numpy(), 2 * want)
    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    owner = b.shard_map(L, E, 2, rank_tokens=counts.cpu().numpy())
    for l in range(L):
        top2 = np.argsort(-want[l], kind="stable")[:2]
        assert owner[l, top2[0]] != owner[l, top2[1]]  # the two hottest experts split
        assert np.bincount(owner[l], minlength=2).tolist() == [4, 4]
    w.close()


@pytest.mark.parametrize("E,k", [(8, 2), (16, 4), (96, 3)])
def test_routing_pair_histogram_and_coselect_map(ctx, E, k):
    """Device co-selection histogram: pairs[l][a][b] (a < b)
    equal a host count of the tokens holding both, accumulate across calls
    (shared-memory counters up to 64 experts, global atomics beyond), and
    feed the co-selection shard map, which never co-locates more
    co-selections than the popularity map."""
    import importlib.util
    import os
    L, n = 3, 777
    rs = np.random.RandomState(E + k)
    host = np.stack([np.stack([rs.choice(E, k, replace=False) for _ in range(n)]) for _ in range(L)]).astype(np.int32)
    ids = torch.tensor(host, device="cuda")
    pairs = torch.zeros((L, E, E), dtype=torch.int64, device="cuda")
    ctx.routing_pair_histogram(ids, pairs)
    ctx.routing_pair_histogram(ids, pairs)
    counts = torch.zeros((L, E), dtype=torch.int64, device="cuda")
    ctx.routing_histogram(ids, counts)
    torch.cuda.synchronize()
    want = np.zeros((L, E, E), np.int64)
    for l in range(L):
        for t in range(n):
            for j1 in range(k):
                for j2 in range(j1 + 1, k):
                    a, b = sorted((host[l, t, j1], host[l, t, j2]))
                    want[l, a, b] += 1
    got = pairs.cpu().numpy()
    assert np.array_equal(got, 2 * want)
    cnt = counts.cpu().numpy()
    owner, _ = M.ep_shard_map_coselect(cnt, got, 2)
    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    lpt = b.shard_map(L, E, 2, rank_tokens=cnt)
    for l in range(L):
        same = lambda o: sum(int(got[l, a, c]) for a in range(E) for c in range(a + 1, E) if o[a] == o[c])
        assert same(owner[l]) <= same(lpt[l])
        assert np.bincount(owner[l], minlength=2).tolist() == [E // 2, E // 2]


def test_fused_sparsity_counters_match_reference_sink(ctx, libopts):
    """Activation-sparsity counters fused into the up-projection epilogues (f2)
    against the reference's sparsity_histogram of its ActivationSink values."""
    ref = O.Reference() if O.reference_available() else None
    if ref is None:
        pytest.skip("oracle/_ref not built")
    thr = [0.001, 0.01, 0.1, 1.0]  # the reference CLI defaults (moe_orch_cli.cpp:412)
    L, E, k, d, f, n = 4, 8, 2, 32, 64, 64
    shape = O.Shape(L, E, k, d, f, 4)
    wref = ref.random_model(shape, 3)
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 4), M.DTYPE_F32)
    w.upload_oracle(wref)
    wd = O.Weights(shape)
    for l in range(L):
        for e in range(E):
            for dst, src in zip(wd.expert(l, e), w.download_expert(l, e)):
                dst[:] = src
        wd.router[l][:] = w.download_router(l)
    toks = np.random.RandomState(0).randn(n, d).astype(np.float32).astype(np.float64)
    sink = ref.model_forward(shape, wd, toks, with_sink=True, sink_cap=n * L * k * f)[4]
    vals = np.abs(sink.reshape(n, L, k, f))
    want = np.array([[int((vals[:, l] < t).sum()) for t in thr] for l in range(L)])
    x = torch.tensor(toks, dtype=torch.float32, device="cuda")
    ids = torch.zeros((L, n, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, n, k), device="cuda")
    counts = torch.zeros((L, len(thr)), dtype=torch.int64, device="cuda")
    w.forward_sparsity(x, ids, g, thr, counts)
    torch.cuda.synchronize()
    got = counts.cpu().numpy()
    assert np.abs(got - want).max() <= 2, (got, want)  # fp32 vs fp64 at the thresholds
    with pytest.raises(M.MoeError) as ei:
        w.forward_sparsity(x, ids, g, [0.1, 0.01], counts)
    assert ei.value.kind == "ValidationError"
    # tcgen05 grouped-GEMM epilogue vs generic kernel at the Mixtral shape
    s = M.Shape(1, 8, 2, 4096, 14336, 2)
    wt = M.Weights(ctx, s, M.DTYPE_BF16)
    libopts(prefill=0)
    wgn = M.Weights(ctx, s, M.DTYPE_BF16)
    libopts(prefill=1)
    assert wt.expert_path(128) == 3 and wgn.expert_path(128) == 2
    xs = torch.randn(128, 4096, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
    res = []
    for ww in (wt, wgn):
        ww.random(4)
        c = torch.zeros((1, len(thr)), dtype=torch.int64, device="cuda")
        ww.forward_sparsity(xs.clone(), torch.zeros((1, 128, 2), dtype=torch.int32, device="cuda"),
                            torch.zeros((1, 128, 2), device="cuda"), thr, c)
        torch.cuda.synchronize()
        res.append(c.cpu().numpy()[0])
    total = 128 * 2 * 14336
    assert res[1][-1] <= total and res[0][-1] > 0
    # bf16 activations (tensor-core operands) vs fp32 ones: counts agree
    # closely (the smallest bucket is the most sensitive to the X rounding)
    assert np.all(np.abs(res[0] - res[1]) <= 0.05 * res[1] + 100), res
    wt.close()
    wgn.close()
    w.close()


def test_x22b_layer_decode_and_prefill_vs_oracle(ctx, orc):
    """Config X shape (Mixtral-8x22B: d=6144, ffn=16384), bf16: batch-1 decode
    through the streaming kernel, a 2-layer stack through the persistent
    kernel (teacher-forced layer 1), and a 96-token prefill through the
    tcgen05 grouped GEMM, each against the fp64 oracle on the device-held
    weights."""
    L, d, f = 2, 6144, 16384
    w = M.Weights(ctx, M.Shape(L, 8, 2, d, f, 2), M.DTYPE_BF16)
    w.random(7)
    assert w.expert_path(1) == 1 and w.expert_path(96) == 3 and w.forward_launches(1) == 1
    rs = np.random.RandomState(7)
    x = f32(rs.randn(d))
    # decode, layer 0
    xd = torch.tensor(x[None], dtype=torch.float32, device="cuda")
    idd = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    gd = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    xo = torch.empty_like(xd)
    w.layer_forward(0, xd, xo, idd, gd)
    torch.cuda.synchronize()
    ids, g, delta, mg = oracle_layer(orc, w, 0, x, 2)
    if mg > 1e-5:
        assert list(idd.cpu().numpy()[0]) == list(ids)
    err = normwise(xo.cpu().numpy()[0].astype(np.float64) - x, delta)
    print(f"X decode normwise error {err:.3e}")
    assert err < 1e-4
    # persistent 2-layer stack; layer 1 teacher-forced on the device's x_1
    xs = torch.tensor(x[None], dtype=torch.float32, device="cuda")
    ids2 = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
    g2 = torch.zeros((L, 1, 2), dtype=torch.float32, device="cuda")
    w.forward(xs, ids2, g2)
    torch.cuda.synchronize()
    x1 = xo.cpu().numpy()[0].astype(np.float64)
    ids1, _, delta1, mg1 = oracle_layer(orc, w, 1, f32(x1), 2)
    if mg1 > 1e-5:
        assert list(ids2.cpu().numpy()[1, 0]) == list(ids1)
    err1 = normwise(xs.cpu().numpy()[0].astype(np.float64) - x1, delta1)
    assert err1 < 1e-3, err1
    # prefill, 96 tokens (tcgen05), sampled tokens vs oracle
    n = 96
    xp = f32(rs.randn(n, d))
    xpd = torch.tensor(xp, dtype=torch.float32, device="cuda")
    xpo = torch.empty_like(xpd)
    idp = torch.zeros((n, 2), dtype=torch.int32, device="cuda")
    gp = torch.zeros((n, 2), dtype=torch.float32, device="cuda")
    w.layer_forward(0, xpd, xpo, idp, gp)
    torch.cuda.synchronize()
    out = xpo.cpu().numpy().astype(np.float64)
    cache = {}
    router = w.download_router(0)
    worst = 0.0
    for t in (0, 37, 95):
        ids_t, g_t, logits = orc.gate_topk(router, xp[t], 2)
        if margin(logits, 2) > 1e-5:
            assert list(idp.cpu().numpy()[t]) == list(ids_t)
        dl = np.zeros(d)
        for e, ge in zip(idp.cpu().numpy()[t], gp.cpu().numpy()[t]):
            if int(e) not in cache:
                cache[int(e)] = w.download_expert(0, int(e))
            dl += ge * orc.expert_ffn(*cache[int(e)], xp[t])
        worst = max(worst, normwise(out[t] - xp[t], dl))
    print(f"X prefill (tcgen05) normwise error {worst:.3e}")
    assert worst < TOL_BF16
    w.close()


@pytest.mark.parametrize("E,k,d,f,dt,n_tok", [
    (16, 4, 1024, 2048, M.DTYPE_BF16, 1),     # streaming decode, k > 2
    (64, 8, 512, 1024, M.DTYPE_BF16, 1),      # many experts, k = 8
    (8, 8, 512, 768, M.DTYPE_F32, 1),         # k == E (every expert selected)
    (1, 1, 256, 512, M.DTYPE_BF16, 1),        # single expert
    (256, 2, 256, 256, M.DTYPE_F32, 3),       # E at the 256 limit, generic multi-token
    (16, 4, 256, 512, M.DTYPE_BF16, 300),     # tcgen05 prefill with k = 4 (ragged experts)
    (8, 2, 256, 512, M.DTYPE_BF16, 2),        # tcgen05 at 2 tokens (tiny N)
])
def test_edge_geometries_vs_oracle(ctx, orc, E, k, d, f, dt, n_tok):
    """Routing geometries beyond Mixtral's (E, k) = (8, 2), through whichever
    kernel the library picks, against the fp64 oracle on device-held values."""
    esz = 2 if dt == M.DTYPE_BF16 else 4
    w = M.Weights(ctx, M.Shape(2, E, k, d, f, esz), dt)
    w.random(E * 31 + k)
    rs = np.random.RandomState(E + k)
    x = f32(rs.randn(n_tok, d))
    xd = torch.tensor(x, dtype=torch.float32, device="cuda")
    xo = torch.empty_like(xd)
    idd = torch.zeros((n_tok, k), dtype=torch.int32, device="cuda")
    gd = torch.zeros((n_tok, k), dtype=torch.float32, device="cuda")
    w.layer_forward(1, xd, xo, idd, gd)
    torch.cuda.synchronize()
    out = xo.cpu().numpy().astype(np.float64)
    ids_dev, g_dev = idd.cpu().numpy(), gd.cpu().numpy()
    router = w.download_router(1)
    tol = TOL_BF16 if (dt == M.DTYPE_BF16 and n_tok > 1) else 1e-4
    cache = {}
    for t in sorted({0, n_tok // 2, n_tok - 1}):
        ids, g, logits = orc.gate_topk(router, x[t], k)
        if margin(logits, k) > 1e-5:
            assert list(ids_dev[t]) == list(ids)
            assert np.abs(g_dev[t] - g).max() < 1e-5
        assert list(ids_dev[t]) == sorted(ids_dev[t])  # ascending ids (model.cpp:96-97)
        assert abs(float(g_dev[t].sum()) - 1.0) < 1e-5
        delta = np.zeros(d)
        for e, ge in zip(ids_dev[t], g_dev[t]):
            if int(e) not in cache:
                cache[int(e)] = w.download_expert(1, int(e))
            delta += ge * orc.expert_ffn(*cache[int(e)], x[t])
        err = normwise(out[t] - x[t], delta)
        assert err < tol, (t, err)
    w.close()


@pytest.mark.parametrize("dt", [M.DTYPE_BF16, M.DTYPE_F32])
def test_layer_forward_batch1_is_one_launch_every_layer(ctx, orc, libopts, dt):
    """moe_layer_forward at batch 1 runs the persistent kernel as a 1-layer
    stack (one launch): every layer index of a 3-layer model against the
    per-layer kernels (router + experts + reduce) and the oracle, out of
    place and in place."""
    L, d, f = 3, 4096, 14336
    s = M.Shape(L, 8, 2, d, f, 2 if dt == M.DTYPE_BF16 else 4)
    w = M.Weights(ctx, s, dt)
    libopts(stack=0)
    w_ref = M.Weights(ctx, s, dt)
    libopts(stack=1)
    assert w.layer_launches(1) == 1 and w_ref.layer_launches(1) == 3
    w.random(21)
    w_ref.random(21)
    rs = np.random.RandomState(4)
    for l in range(L):
        x = f32(0.5 * rs.randn(d))
        outs = []
        for ww, inplace in ((w, False), (w, True), (w_ref, False)):
            xd = torch.tensor(x[None], dtype=torch.float32, device="cuda")
            xo = xd if inplace else torch.empty_like(xd)
            ids = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
            g = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
            ww.layer_forward(l, xd, xo, ids, g)
            torch.cuda.synchronize()
            outs.append((xo.cpu().numpy()[0].astype(np.float64), ids.cpu().numpy()[0], g.cpu().numpy()[0]))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
        oid, og, delta, mg = oracle_layer(orc, w, l, x, 2)
        if mg > 1e-5:
            assert list(outs[0][1]) == list(oid) == list(outs[2][1]), l
            assert np.abs(outs[0][2] - og).max() < 1e-5
        err = normwise(outs[0][0] - x, delta)
        assert err < (1e-4 if dt == M.DTYPE_BF16 else TOL_F32), (l, err)
        assert normwise(outs[0][0] - x, outs[2][0] - x) < 1e-5
    w.close()
    w_ref.close()


@pytest.mark.parametrize("dt", [M.DTYPE_BF16, M.DTYPE_F32])
def test_one_layer_model_runs_the_single_barrier_kernel(ctx, orc, libopts, dt):
    """A 1-layer model (BASELINE configs[1] as its own model) gets the same
    one-launch single-barrier kernel at batch 1 for moe_layer_forward and
    moe_forward — it has no next router, so no projections are needed — and
    matches the oracle and the per-layer kernels."""
    d, f = 4096, 14336
    s = M.Shape(1, 8, 2, d, f, 2 if dt == M.DTYPE_BF16 else 4)
    w = M.Weights(ctx, s, dt)
    libopts(stack=0)
    w_ref = M.Weights(ctx, s, dt)
    libopts(stack=1)
    assert w.layer_launches(1) == 1 and w.forward_launches(1) == 1 and w_ref.layer_launches(1) == 3
    w.random(23)
    w_ref.random(23)
    rs = np.random.RandomState(6)
    for rep in range(3):
        x = f32(0.5 * rs.randn(d))
        outs = []
        for ww, fwd in ((w, False), (w, True), (w_ref, False)):
            xd = torch.tensor(x[None], dtype=torch.float32, device="cuda")
            ids = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
            g = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
            if fwd:
                xo = xd
                ww.forward(xd, ids.view(1, 1, 2), g.view(1, 1, 2))
            else:
                xo = torch.empty_like(xd)
                ww.layer_forward(0, xd, xo, ids, g)
            torch.cuda.synchronize()
            outs.append((xo.cpu().numpy()[0].astype(np.float64), ids.cpu().numpy()[0], g.cpu().numpy()[0]))
        assert all(np.array_equal(outs[0][i], outs[1][i]) for i in range(3)), rep  # same kernel, same launch
        oid, og, delta, mg = oracle_layer(orc, w, 0, x, 2)
        if mg > 1e-5:
            assert list(outs[0][1]) == list(oid) == list(outs[2][1]), rep
            assert np.abs(outs[0][2] - og).max() < 1e-5
        err = normwise(outs[0][0] - x, delta)
        assert err < (1e-4 if dt == M.DTYPE_BF16 else TOL_F32), (rep, err)
        assert normwise(outs[0][0] - x, outs[2][0] - x) < 1e-5
    w.close()
    w_ref.close()
