"""Per-CTA stream-end spread of the persistent stack kernel from a trace
(the slow SMs and the per-layer spread).

    python tools/spread_analysis.py
"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch
import paper_2402_07033_b200 as M
from trace_stack import to_ns
ctx = M.Ctx(0)
L = 32
w = M.Weights(ctx, M.Shape(L, 8, 2, 4096, 14336, 2), M.DTYPE_BF16)
w.random(0)
x = torch.randn(1, 4096, device="cuda")
ids = torch.zeros((L, 1, 2), dtype=torch.int32, device="cuda")
g = torch.zeros((L, 1, 2), device="cuda")
for _ in range(3):
    w.forward(x, ids, g)
torch.cuda.synchronize()
ends = []
smids = []
for rep in range(4):
    raw = w.debug_trace_forward(x, ids, g).copy()
    t, ghz = to_ns(raw)
    smids.append(raw[1, :, 13].astype(int).copy())
    # per layer: stream duration per CTA (first stage landed -> stream done)
    dur = t[1:L-1, :, 2] - t[1:L-1, :, 1]
    endrel = t[1:L-1, :, 2] - np.median(t[1:L-1, :, 2], axis=1, keepdims=True)
    ends.append((dur, endrel))
dur, endrel = ends[-1]
print("smid mapping stable across launches:", all(np.array_equal(smids[0], s) for s in smids))
m = endrel.mean(axis=0)
print("per-CTA mean end offset vs median (us): min %.2f max %.2f std %.2f" % (m.min()/1e3, m.max()/1e3, m.std()/1e3))
# correlation of per-CTA offsets between even and odd layers
a = endrel[0::2].mean(axis=0); b = endrel[1::2].mean(axis=0)
print("corr(even layers, odd layers) of per-CTA end offset: %.3f" % np.corrcoef(a, b)[0, 1])
a2 = ends[0][1].mean(axis=0)
print("corr(launch 0, launch 3): %.3f" % np.corrcoef(a2, m)[0, 1])
dm = dur.mean(axis=0)
print("stream duration per CTA (us): min %.1f median %.1f max %.1f" % (dm.min()/1e3, np.median(dm)/1e3, dm.max()/1e3))
order = np.argsort(-m)
print("slowest CTAs:", [(int(c), int(smids[-1][c]), round(m[c]/1e3, 2)) for c in order[:12]])
print("fastest CTAs:", [(int(c), int(smids[-1][c]), round(m[c]/1e3, 2)) for c in order[-6:]])
# start offsets (first stage landed)
st = t[1:L-1, :, 1] - np.median(t[1:L-1, :, 1], axis=1, keepdims=True)
print("start offset std (us) %.2f, corr(start, end) %.3f" % (st.mean(0).std()/1e3, np.corrcoef(st.mean(0), m)[0,1]))
