"""Expert-parallel sharding on ONE GPU with virtual ranks.

W contexts on the same device each take a (world, rank) without a
communicator (moe_ctx_set_virtual_rank).  Each allocates only the experts the
popularity shard map gives its rank, and computes only its partial.  Summing
the W partial deltas must reproduce the unsharded layer: the decode
(streaming kernel), tcgen05 prefill and generic paths all skip remote experts
and zero their rows.  The all-reduce itself (NCCL) is the only piece not
exercised here; it needs >1 GPU.
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


def normwise(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape,dtype,n_tok,tol", [
    ((1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16, 1, 1e-5),    # streaming decode kernel
    ((1, 8, 2, 256, 512, 2), M.DTYPE_BF16, 96, 1e-5),      # tcgen05 prefill
    ((1, 8, 2, 48, 80, 4), M.DTYPE_F32, 5, 1e-5),          # generic kernels
])
def test_virtual_ranks_sum_to_unsharded_layer(gpu, world, shape, dtype, n_tok, tol):
    L, E = shape[0], shape[1]
    owner = _bench().shard_map(L, E, world)
    s = M.Shape(*shape)
    base_ctx = M.Ctx(0)
    full = M.Weights(base_ctx, s, dtype)
    full.random(21)
    x = torch.randn(n_tok, s.hidden_dim, device="cuda")
    ids = torch.zeros((n_tok, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((n_tok, 2), device="cuda")
    want = torch.empty_like(x)
    full.layer_forward(0, x, want, ids, g)
    torch.cuda.synchronize()
    x64 = x.cpu().numpy().astype(np.float64)
    delta_want = want.cpu().numpy().astype(np.float64) - x64

    delta = np.zeros_like(x64)
    owned_bytes = 0
    for r in range(world):
        ctx = M.Ctx(0)
        ctx.set_virtual_rank(world, r)
        w = M.Weights(ctx, s, dtype, owner=owner)
        w.random(21)  # counter-based init: identical values for the owned experts
        owned_bytes += w.device_bytes
        out = torch.empty_like(x)
        ids_r = torch.zeros_like(ids)
        g_r = torch.zeros_like(g)
        w.layer_forward(0, x, out, ids_r, g_r)
        torch.cuda.synchronize()
        assert torch.equal(ids_r, ids)  # every rank routes identically
        delta += out.cpu().numpy().astype(np.float64) - x64
        w.close()
        ctx.close()
    assert normwise(delta, delta_want) < tol
    # each rank holds only its share of the experts (router replicated)
    assert owned_bytes < full.device_bytes * (1.0 + (world - 1) * 0.02)
    full.close()
    base_ctx.close()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape,dtype,n_tok,tol", [
    ((1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16, 1, 1e-5),    # streaming decode kernel
    ((1, 8, 2, 256, 1024, 2), M.DTYPE_BF16, 96, 1e-5),     # tcgen05 prefill (f/world % 128 == 0)
    ((1, 8, 2, 48, 80, 4), M.DTYPE_F32, 5, 1e-5),          # generic kernels
])
def test_tensor_parallel_virtual_ranks_sum_to_unsharded_layer(gpu, world, shape, dtype, n_tok, tol):
    """Tensor parallelism: each rank holds ffn rows [r*f/W, (r+1)*f/W) of every
    expert; the ranks' partial deltas sum to the unsharded layer, and the
    ranks' weight slices reassemble the unsharded model's experts exactly."""
    s = M.Shape(*shape)
    base_ctx = M.Ctx(0)
    full = M.Weights(base_ctx, s, dtype)
    full.random(21)
    x = torch.randn(n_tok, s.hidden_dim, device="cuda")
    ids = torch.zeros((n_tok, 2), dtype=torch.int32, device="cuda")
    g = torch.zeros((n_tok, 2), device="cuda")
    want = torch.empty_like(x)
    full.layer_forward(0, x, want, ids, g)
    torch.cuda.synchronize()
    x64 = x.cpu().numpy().astype(np.float64)
    delta_want = want.cpu().numpy().astype(np.float64) - x64
    e_chk = int(ids[0, 0])
    wi_full, wg_full, wo_full = full.download_expert(0, e_chk)
    wi, wg, wo = (np.full_like(m, np.nan) for m in (wi_full, wg_full, wo_full))

    delta = np.zeros_like(x64)
    for r in range(world):
        ctx = M.Ctx(0)
        ctx.set_virtual_rank(world, r)
        w = M.Weights(ctx, s, dtype, tp=True)
        assert w.tp == (world, r, s.ffn_dim // world)
        w.random(21)
        out = torch.empty_like(x)
        ids_r = torch.zeros_like(ids)
        g_r = torch.zeros_like(g)
        w.layer_forward(0, x, out, ids_r, g_r)
        torch.cuda.synchronize()
        assert torch.equal(ids_r, ids)
        delta += out.cpu().numpy().astype(np.float64) - x64
        f0, f1 = r * s.ffn_dim // world, (r + 1) * s.ffn_dim // world
        a, b, c = (np.full_like(m, np.nan) for m in (wi_full, wg_full, wo_full))
        from paper_2402_07033_b200 import capi  # download into full-size buffers
        capi.check(capi.lib().moe_weights_download_expert(w.h, 0, e_chk, capi._dptr(a), capi._dptr(b),
                                                           capi._dptr(c)))
        wi[f0:f1], wg[f0:f1], wo[:, f0:f1] = a[f0:f1], b[f0:f1], c[:, f0:f1]
        assert np.isnan(a[:f0]).all() and np.isnan(c[:, f1:]).all()  # only the slice is written
        w.close()
        ctx.close()
    assert np.array_equal(wi, wi_full) and np.array_equal(wg, wg_full) and np.array_equal(wo, wo_full)
    assert normwise(delta, delta_want) < tol
    full.close()
    base_ctx.close()
