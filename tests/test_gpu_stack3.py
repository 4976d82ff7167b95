"""decode_stack3_kernel (stack_kernel=3: up rows first, the next layer's
routing resolved by the producer during the down phase) against
decode_stack2_kernel on the same weights.

Both kernels split the same rows over the same CTAs, do the same per-row
fp32 arithmetic and sum the partials in 64-bit fixed point, so x_L, every
layer's ids, gates and router logits must be BIT-identical — across repeated
launches (barrier/route counters and the accumulator rotation carry over),
shrunk grids (more rows per CTA in smem), fp32 and bf16, and k = 1..3.
The oracle anchor of the stack path itself is test_gpu_parity_full.py::S and
test_gpu_parity.py (they run whichever kernel is the default).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_07033_b200 as M  # noqa: E402
from _parity import normwise, oracle_route  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()
    c = M.Ctx(0)
    yield c
    c.close()


def _run(w, kern, x0, L, E, k, libopts, launches=3):
    libopts(stack_kernel=kern)
    outs = []
    for _ in range(launches):
        x = torch.tensor(x0[None], dtype=torch.float32, device="cuda")
        ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, 1, k), dtype=torch.float32, device="cuda")
        lg = torch.zeros((L, E), dtype=torch.float32, device="cuda")
        w.forward_logits(x, ids, g, lg)
        torch.cuda.synchronize()
        outs.append(tuple(t.cpu().numpy().copy() for t in (x, ids, g, lg)))
    # graph path (forward) too
    x = torch.tensor(x0[None], dtype=torch.float32, device="cuda")
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, k), dtype=torch.float32, device="cuda")
    w.forward(x, ids, g)
    torch.cuda.synchronize()
    outs.append((x.cpu().numpy(), ids.cpu().numpy(), g.cpu().numpy(), outs[0][3]))
    return outs


@pytest.mark.parametrize("L,E,k,d,f,dt,grid", [
    (6, 8, 2, 4096, 14336, M.DTYPE_BF16, 0),     # Mixtral layers
    (6, 8, 2, 4096, 14336, M.DTYPE_BF16, 74),    # 2x the rows per CTA
    (4, 8, 2, 6144, 16384, M.DTYPE_BF16, 0),     # 8x22B layers
    (5, 8, 1, 1024, 2816, M.DTYPE_BF16, 0),      # top-1
    (5, 6, 3, 1024, 1536, M.DTYPE_BF16, 0),      # E=6, top-3
    (4, 8, 2, 512, 1792, M.DTYPE_F32, 0),        # fp32 mode (config T shape)
    (3, 4, 2, 256, 704, M.DTYPE_F32, 16),        # tiny, CTAs with no rows of a layer
])
def test_stack3_bit_identical_to_stack2(ctx, libopts, L, E, k, d, f, dt, grid):
    if grid:
        libopts(stack_grid=grid)
    s = M.Shape(L, E, k, d, f, 2 if dt == M.DTYPE_BF16 else 4)
    w = M.Weights(ctx, s, dt)
    w.random(5)
    assert w.forward_launches(1) == 1
    x0 = (0.1 * np.random.RandomState(L + d).randn(d)).astype(np.float32).astype(np.float64)
    o2 = _run(w, 2, x0, L, E, k, libopts)
    o3 = _run(w, 3, x0, L, E, k, libopts)
    # stack 3 really ran: only it stamps the producer's globaltimer (slot 13)
    tr = w.debug_trace_forward(torch.tensor(x0[None], dtype=torch.float32, device="cuda"),
                               torch.zeros((L, 1, k), dtype=torch.int32, device="cuda"),
                               torch.zeros((L, 1, k), dtype=torch.float32, device="cuda"))
    assert (tr[0, :(grid or ctx.sm_count), 13] != 0).all()
    for a, b in zip(o2 + o3[:1], o3 + o2[:1]):
        for i, name in enumerate(("x", "ids", "gates", "logits")):
            assert np.array_equal(a[i], b[i]), name
    assert np.isfinite(o3[0][0]).all()
    # the routing the kernel committed is the top-k of the logits it recorded
    lg = o3[0][3].astype(np.float64)
    for l in range(L):
        srt = np.sort(lg[l])[::-1]
        if k < E and (srt[k - 1] - srt[k]) / np.abs(lg[l]).max() > 1e-5:
            assert sorted(np.argsort(-lg[l], kind="stable")[:k]) == list(o3[0][1][l, 0])
    w.close()


def test_stack3_first_layer_routing_vs_oracle(ctx, orc, libopts):
    """Layer 0 of stack 3 against the oracle gate_topk on the downloaded router."""
    libopts(stack_kernel=3)
    L, E, k, d, f = 3, 8, 2, 4096, 14336
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(2)
    x0 = (0.1 * np.random.RandomState(9).randn(d)).astype(np.float32).astype(np.float64)
    x = torch.tensor(x0[None], dtype=torch.float32, device="cuda")
    ids = torch.zeros((L, 1, k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, 1, k), dtype=torch.float32, device="cuda")
    lg = torch.zeros((L, E), dtype=torch.float32, device="cuda")
    w.forward_logits(x, ids, g, lg)
    torch.cuda.synchronize()
    oid, og, olog, marg = oracle_route(orc, w.download_router(0), x0, k)
    assert normwise(lg.cpu().numpy()[0], olog[0]) < 1e-5
    if marg[0] > 1e-5:
        assert list(ids.cpu().numpy()[0, 0]) == list(oid[0])
        assert np.abs(g.cpu().numpy()[0, 0] - og[0]).max() < 1e-5
    w.close()
