"""moe_forward_host_async / moe_host_wait: the pipelined host-buffer steps
equal the device-pointer calls bit for bit (one layer: moe_layer_forward;
whole stack: moe_forward), with several calls in flight over the two staging
slots, including batch 1, prefill and a token count that grows mid-sequence."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_07033_b200 as M  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()
    c = M.Ctx(0)
    yield c
    c.close()


def _device_layer(w, layer, x, k):
    xd = torch.tensor(x, device="cuda")
    xo = torch.empty_like(xd)
    ids = torch.zeros((x.shape[0], k), dtype=torch.int32, device="cuda")
    g = torch.zeros((x.shape[0], k), device="cuda")
    w.layer_forward(layer, xd, xo, ids, g)
    torch.cuda.synchronize()
    return xo.cpu().numpy(), ids.cpu().numpy(), g.cpu().numpy()


def _device_stack(w, x, L, k):
    xd = torch.tensor(x, device="cuda")
    ids = torch.zeros((L, x.shape[0], k), dtype=torch.int32, device="cuda")
    g = torch.zeros((L, x.shape[0], k), device="cuda")
    w.forward(xd, ids, g)
    torch.cuda.synchronize()
    return xd.cpu().numpy(), ids.cpu().numpy(), g.cpu().numpy()


@pytest.mark.parametrize("d,f,dt", [(4096, 14336, M.DTYPE_BF16), (512, 1792, M.DTYPE_F32)])
def test_host_async_layer_and_stack_equal_device_calls(ctx, d, f, dt):
    L, E, k = 3, 8, 2
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2 if dt == M.DTYPE_BF16 else 4), dt)
    w.random(4)
    rs = np.random.RandomState(0)
    calls = []
    for layer, n in [(0, 512), (1, 1), (2, 37), (-1, 1), (-1, 96), (0, 700), (1, 512)]:
        x = (0.1 * rs.randn(n, d)).astype(np.float32)
        nl = L if layer < 0 else 1
        xh = torch.tensor(x).pin_memory()
        out = torch.empty((n, d)).pin_memory()
        ids = torch.empty((nl, n, k) if layer < 0 else (n, k), dtype=torch.int32).pin_memory()
        g = torch.empty(ids.shape).pin_memory()
        t = w.forward_host_async(layer, xh, out, ids, g)
        # the pinned input stays referenced until the wait: freed, torch's
        # caching host allocator would hand its block to the next
        # pin_memory() while the H2D is still queued
        calls.append((t, layer, x, xh, out, ids, g))
    w.host_wait(calls[3][0])  # a middle ticket first
    w.host_wait()
    for t, layer, x, _, out, ids, g in calls:
        want = _device_layer(w, layer, x, k) if layer >= 0 else _device_stack(w, x, L, k)
        assert np.array_equal(out.numpy(), want[0]), (t, layer, float(np.abs(out.numpy() - want[0]).max()))
        assert np.array_equal(ids.numpy(), want[1]), (t, layer)
        assert np.array_equal(g.numpy(), want[2]), (t, layer)
    w.close()


def test_host_async_errors(ctx):
    w = M.Weights(ctx, M.Shape(2, 8, 2, 512, 1792, 4), M.DTYPE_F32)
    x = np.zeros((4, 512), np.float32)
    with pytest.raises(M.MoeError):
        w.forward_host_async(2, x, x.copy(), np.zeros((4, 2), np.int32), np.zeros((4, 2), np.float32))
    w.host_wait()  # nothing in flight: returns
    w.close()


def test_host_async_results_land_in_ticket_order(ctx):
    """Waiting on a batch-1 step (copies on the compute stream) also covers
    the multi-token steps before it (copies on the copy streams), and the
    other way round."""
    L, E, k, d, f = 2, 8, 2, 512, 1792
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 4), M.DTYPE_F32)
    w.random(5)
    rs = np.random.RandomState(3)
    for seq in ([(0, 900), (1, 1)], [(1, 1), (0, 1), (1, 640)], [(0, 333), (-1, 1), (1, 2), (0, 1)]):
        calls = []
        for layer, n in seq:
            x = (0.1 * rs.randn(n, d)).astype(np.float32)
            nl = L if layer < 0 else 1
            out = torch.empty((n, d)).pin_memory()
            ids = torch.empty((nl, n, k) if layer < 0 else (n, k), dtype=torch.int32).pin_memory()
            g = torch.empty(ids.shape).pin_memory()
            xh = torch.tensor(x).pin_memory()  # stays referenced until the wait
            t = w.forward_host_async(layer, xh, out, ids, g)
            calls.append((layer, x, xh, out, ids, g))
        w.host_wait(t)  # the last ticket only
        for layer, x, _, out, ids, g in calls:
            want = _device_layer(w, layer, x, k) if layer >= 0 else _device_stack(w, x, L, k)
            assert np.array_equal(out.numpy(), want[0]), (seq, layer)
            assert np.array_equal(ids.numpy(), want[1]), (seq, layer)
    w.close()
