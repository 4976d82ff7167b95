"""RoutingTrace JSONL emission: the emitter's output is
accepted by the REFERENCE's own loader/validator (trace.cpp:110-141) and
carries the reference model_forward's trace; on the GPU the step is built
from the device routing record (moe_routing_trace_step)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2402_07033_b200 import trace as T


def _ref():
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    return O.Reference()


def test_emitter_round_trips_through_reference_loader(tmp_path):
    ref = _ref()
    shape = O.Shape(4, 8, 2, 32, 64, 8)
    w = ref.random_model(shape, 3)
    rs = np.random.RandomState(0)
    steps = []
    for n in (6, 1, 1):  # one prefill step, two decode steps
        toks = rs.randn(n, 32)
        out, cnt, gate, kind = ref.model_forward(shape, w, toks)[:4]
        assert kind == (1 if n == 1 else 0)
        steps.append(T.step_from_counts(cnt.reshape(4, 8), gate.reshape(4, 8), n))
    path = str(tmp_path / "t.jsonl")
    T.save_trace_jsonl(steps, path)
    assert ref.load_trace_jsonl(path, shape) == 3
    line = open(path).readline()
    assert line.startswith('{"kind":"prefill","layers":[[[')
    # a corrupted count is rejected by the reference validator
    bad = steps[1]["layers"][0][0]
    bad[1] = 2
    T.save_trace_jsonl(steps, path)
    with pytest.raises(ValueError, match="ValidationError"):
        ref.load_trace_jsonl(path, shape)


@pytest.mark.gpu
def test_device_trace_step_matches_reference(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2402_07033_b200 as M

    ref = _ref()
    orc_shape = O.Shape(4, 8, 2, 32, 64, 4)
    wref = ref.random_model(orc_shape, 3)
    ctx = M.Ctx(0)
    w = M.Weights(ctx, M.Shape(4, 8, 2, 32, 64, 4), M.DTYPE_F32)
    w.upload_oracle(wref)
    rs = np.random.RandomState(1)
    steps = []
    for n in (6, 1):
        toks = rs.randn(n, 32).astype(np.float32).astype(np.float64)
        # the reference on the device-held (fp32-rounded) weights
        wd = O.Weights(orc_shape)
        for l in range(4):
            for e in range(8):
                for dst, src in zip(wd.expert(l, e), w.download_expert(l, e)):
                    dst[:] = src
            wd.router[l][:] = w.download_router(l)
        _, cnt, gate, kind = ref.model_forward(orc_shape, wd, toks)[:4]
        x = torch.tensor(toks, dtype=torch.float32, device="cuda")
        ids = torch.zeros((4, n, 2), dtype=torch.int32, device="cuda")
        g = torch.zeros((4, n, 2), device="cuda")
        w.forward(x, ids, g)
        torch.cuda.synchronize()
        st = T.device_step(ctx, ids, g, 8)
        want = T.step_from_counts(cnt.reshape(4, 8), gate.reshape(4, 8), n)
        assert st["kind"] == want["kind"]
        for a, b in zip(st["layers"], want["layers"]):
            assert [s[:2] for s in a] == [s[:2] for s in b]  # experts + token counts exact
            assert np.allclose([s[2] for s in a], [s[2] for s in b], rtol=0, atol=1e-6)
        steps.append(st)
    path = str(tmp_path / "gpu.jsonl")
    T.save_trace_jsonl(steps, path)
    assert ref.load_trace_jsonl(path, orc_shape) == 2
    w.close()
    ctx.close()
