"""The fused prefill layer (router with dispatch bases -> one grouped tcgen05
kernel that scatters the rows, runs both GEMMs and writes x + the combined
expert outputs) against the unfused chain (router, permute, gather, grouped
kernel, combine_k2) on the same weights.

Same routing kernel arithmetic, same stable permutation, same GEMM tiles and
the same combine adds in the same order, so outputs, ids and gates must be
BIT-identical; the oracle anchor of the prefill path is
test_gpu_parity_full.py::P and test_gpu_parity.py (they run the default,
fused, path).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_07033_b200 as M  # noqa: E402
from _parity import f32, normwise  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()
    c = M.Ctx(0)
    yield c
    c.close()


def _layer(w, x, k, reps=2):
    outs = []
    for _ in range(reps):
        xd = torch.tensor(x, dtype=torch.float32, device="cuda")
        xo = torch.full_like(xd, float("nan"))
        ids = torch.full((x.shape[0], k), -1, dtype=torch.int32, device="cuda")
        g = torch.zeros((x.shape[0], k), dtype=torch.float32, device="cuda")
        w.layer_forward(0, xd, xo, ids, g)
        torch.cuda.synchronize()
        outs.append((xo.cpu().numpy(), ids.cpu().numpy(), g.cpu().numpy()))
    assert all(np.array_equal(outs[0][i], o[i]) for o in outs[1:] for i in range(3)), "not deterministic"
    return outs[0]


@pytest.mark.parametrize("E,k,d,f,n_tok", [
    (8, 2, 4096, 14336, 512),    # configs[2]
    (8, 2, 4096, 14336, 96),     # small experts
    (8, 2, 4096, 14336, 1537),   # > 256 tokens per expert: several chunks, ragged block
    (8, 2, 1024, 2048, 3),       # fewer tokens than a router block
    (8, 1, 1024, 2048, 333),     # top-1
    (6, 3, 1024, 1536, 200),     # E = 6, top-3
    (16, 4, 1024, 1024, 700),    # E = 16, top-4
    (8, 2, 6144, 16384, 300),    # 8x22B layer
])
def test_fused_prefill_bit_identical_to_unfused(ctx, libopts, E, k, d, f, n_tok):
    s = M.Shape(1, E, k, d, f, 2)
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    w.random(3)
    assert w.expert_path(n_tok) == 3
    x = f32(np.random.RandomState(n_tok).randn(n_tok, d))
    libopts(prefill_fused=1)
    assert w.forward_launches(n_tok) == 3
    fused = _layer(w, x, k)
    libopts(prefill_fused=0)
    assert w.forward_launches(n_tok) > 3
    ref = _layer(w, x, k)
    for i, name in enumerate(("x_out", "ids", "gates")):
        assert np.array_equal(fused[i], ref[i]), name
    assert np.isfinite(fused[0]).all()
    w.close()


def test_fused_prefill_multilayer_forward_and_inplace(ctx, libopts):
    """A 3-layer forward (x in place, layers chained through the fused
    kernels) equals the unfused chain bit for bit, ids of every layer too."""
    L, E, k, d, f, n = 3, 8, 2, 1024, 2048, 640
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(8)
    x0 = 0.1 * f32(np.random.RandomState(1).randn(n, d))
    res = {}
    for fused in (1, 0):
        libopts(prefill_fused=fused)
        x = torch.tensor(x0, dtype=torch.float32, device="cuda")
        ids = torch.zeros((L, n, k), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, n, k), dtype=torch.float32, device="cuda")
        w.forward(x, ids, g)
        torch.cuda.synchronize()
        res[fused] = (x.cpu().numpy(), ids.cpu().numpy(), g.cpu().numpy())
    for i in range(3):
        assert np.array_equal(res[1][i], res[0][i])
    assert normwise(res[1][0] - x0, res[0][0] - x0) == 0.0
    w.close()
