"""compute-sanitizer workload: the fused prefill layer and forward (ragged
token counts, top-2 / top-3), stack kernels 2 and 3 and the 1-layer stack,
and the pipelined host-buffer API, at small shapes (the sanitizer slows
kernels 10-100x).

    compute-sanitizer --tool memcheck  python tools/sanitize_workload.py
    compute-sanitizer --tool racecheck python tools/sanitize_workload.py
    compute-sanitizer --tool synccheck python tools/sanitize_workload.py
    compute-sanitizer --tool initcheck python tools/sanitize_workload.py
"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2402_07033_b200 as M
ctx = M.Ctx(0)
for (E, k, d, f, n) in [(8, 2, 1024, 2048, 37), (6, 3, 1024, 1536, 20)]:
    w = M.Weights(ctx, M.Shape(2, E, k, d, f, 2), M.DTYPE_BF16); w.random(3)
    x = torch.tensor(np.random.RandomState(n).randn(n, d).astype(np.float32), device="cuda")
    xo = torch.empty_like(x); ids = torch.zeros((n, k), dtype=torch.int32, device="cuda"); g = torch.zeros((n, k), device="cuda")
    w.layer_forward(0, x, xo, ids, g); torch.cuda.synchronize()
    xx = x.clone(); ids2 = torch.zeros((2, n, k), dtype=torch.int32, device="cuda"); g2 = torch.zeros((2, n, k), device="cuda")
    w.forward(xx, ids2, g2); torch.cuda.synchronize()
    w.close()
# stack 2/3 + 1-layer stack, small
for kern in (2, 3):
    M.set_option("stack_kernel", kern)
    w = M.Weights(ctx, M.Shape(3, 8, 2, 1024, 2048, 2), M.DTYPE_BF16); w.random(1)
    x = 0.1 * torch.randn(1, 1024, device="cuda"); ids = torch.zeros((3, 1, 2), dtype=torch.int32, device="cuda"); g = torch.zeros((3, 1, 2), device="cuda")
    w.forward(x, ids, g); torch.cuda.synchronize()
    xo = torch.empty_like(x); w.layer_forward(1, x, xo, ids[0], g[0]); torch.cuda.synchronize()
    w.close()
# pipelined host-buffer API: batch 1 (copies on the compute stream) and
# multi-token (copy streams), one layer and the whole stack
w = M.Weights(ctx, M.Shape(2, 8, 2, 1024, 2048, 2), M.DTYPE_BF16); w.random(2)
keep = []
for layer, n in [(0, 1), (1, 40), (-1, 1), (-1, 9)]:
    nl = 2 if layer < 0 else 1
    xh = (0.1 * torch.randn(n, 1024)).pin_memory(); out = torch.empty(n, 1024).pin_memory()
    ih = torch.empty((nl, n, 2) if layer < 0 else (n, 2), dtype=torch.int32).pin_memory(); gh = torch.empty(ih.shape).pin_memory()
    keep.append((xh, out, ih, gh)); w.forward_host_async(layer, xh, out, ih, gh)
w.host_wait(); w.close()
print("sanitizer workload done")
