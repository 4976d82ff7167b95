"""One moe_weights used from several CUDA streams (the scratch,
the persistent kernels' barrier words and the captured graphs are per
weights).  Calls on different streams are ordered by the library
(capi_internal.h StreamOrder), so back-to-back calls on alternating streams with no
host synchronisation give the serial results bit for bit — for the batch-1
persistent stack kernel, the per-layer decode path and the multi-token
(tcgen05 prefill) path.
"""
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


@pytest.mark.parametrize("n_tok", [1, 96])
def test_alternating_streams_equal_serial(ctx, n_tok):
    L, E, k, d, f = 4, 8, 2, 512, 1024
    w = M.Weights(ctx, M.Shape(L, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(5)
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(3)
    inputs = [(0.3 * torch.randn(n_tok, d, generator=g)).to(dev) for _ in range(6)]

    def run(x, stream=None):
        ids = torch.empty(L * n_tok * k, dtype=torch.int32, device=dev)
        gates = torch.empty(L * n_tok * k, dtype=torch.float32, device=dev)
        w.forward(x, ids, gates, stream=stream)
        return x, ids, gates

    serial = []
    for x in inputs:
        y = x.clone()
        run(y)
        torch.cuda.synchronize()
        serial.append(y.cpu())

    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    for rep in range(3):
        outs = []
        for i, x in enumerate(inputs):
            s = streams[(i + rep) % len(streams)]
            with torch.cuda.stream(s):
                y = x.clone()
            s.synchronize()  # only the clone; the forwards themselves are not waited on
            outs.append(run(y, stream=s.cuda_stream)[0])
        torch.cuda.synchronize()
        for i, y in enumerate(outs):
            assert torch.equal(y.cpu(), serial[i]), (rep, i)
    w.close()


def test_layer_forward_alternating_streams(ctx):
    """moe_layer_forward (router + experts + combine into x_out) on two
    streams back to back, 1 and 40 tokens."""
    E, k, d, f = 8, 2, 512, 1024
    w = M.Weights(ctx, M.Shape(2, E, k, d, f, 2), M.DTYPE_BF16)
    w.random(9)
    dev = torch.device("cuda:0")
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for n in (1, 40):
        x = 0.3 * torch.randn(n, d, device=dev)
        torch.cuda.synchronize()
        want = []
        for layer in (0, 1):
            o = torch.empty_like(x)
            ids = torch.empty(n * k, dtype=torch.int32, device=dev)
            gts = torch.empty(n * k, dtype=torch.float32, device=dev)
            w.layer_forward(layer, x, o, ids, gts)
            torch.cuda.synchronize()
            want.append(o.clone())
        bufs = [(layer, torch.empty_like(x), torch.empty(n * k, dtype=torch.int32, device=dev),
                 torch.empty(n * k, dtype=torch.float32, device=dev))
                for rep in range(4) for layer in (0, 1)]
        torch.cuda.synchronize()
        got = []
        for i, (layer, o, ids, gts) in enumerate(bufs):  # no host waits in between
            s = s1 if i % 2 else s2
            w.layer_forward(layer, x, o, ids, gts, stream=s.cuda_stream)
            got.append((layer, o))
        torch.cuda.synchronize()
        for layer, o in got:
            assert torch.equal(o, want[layer])
    w.close()
