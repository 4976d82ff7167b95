"""The expert-parallel code path WITH its NCCL exchange, on one GPU.

With the debug option force_ep=1 a world-size-1 context still builds a (1-rank) NCCL
communicator.  It then takes the EP path: local partials → reduce →
ncclAllReduce (captured in the CUDA graph for batch-1 decode) → residual +
next-layer router.  The outputs must match the single-GPU persistent stack
kernel.  This exercises the dlopen'ed NCCL, graph capture of the collective
and the per-layer EP orchestration on real hardware.  Only the multi-rank
all-reduce itself needs more than one GPU.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_07033_b200 as M  # noqa: E402


def normwise(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


@pytest.mark.parametrize("n_tok", [1, 64])
def test_forced_ep_path_matches_single_gpu(gpu, libopts, n_tok):
    L = 4
    s = M.Shape(L, 8, 2, 1024, 2048, 2)
    ref_ctx = M.Ctx(0)
    ref = M.Weights(ref_ctx, s, M.DTYPE_BF16)
    ref.random(9)
    libopts(force_ep=1)
    ctx = M.Ctx(0)
    ctx.init_ep(1, 0, M.Ctx.unique_id())
    w = M.Weights(ctx, s, M.DTYPE_BF16)
    w.random(9)
    if n_tok == 1:
        assert w.forward_launches(1) == 1 + 3 * L  # decode + reduce + residual/router per layer
        assert ref.forward_launches(1) == 1        # stack kernel
    x0 = torch.randn(n_tok, 1024, device="cuda")
    outs = []
    for ww in (ref, w):
        x = x0.clone()
        ids = torch.zeros((L, n_tok, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((L, n_tok, 2), device="cuda")
        for _ in range(2):  # second call replays the captured graph (with the collective)
            x.copy_(x0)
            ww.forward(x, ids, g)
        torch.cuda.synchronize()
        outs.append((x.cpu().numpy().astype(np.float64), ids.cpu().numpy()))
    (xr, idr), (xe, ide) = outs
    assert np.array_equal(idr, ide)
    x0n = x0.cpu().numpy().astype(np.float64)
    assert normwise(xe - x0n, xr - x0n) < 1e-4
    w.close()
    ctx.close()
    ref.close()
    ref_ctx.close()
