cat > /tmp/pf1.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2402_07033_b200 as M
fused = int(sys.argv[1])
M.set_option("prefill_fused", fused)
ctx = M.Ctx(0); w = M.Weights(ctx, M.Shape(1, 8, 2, 4096, 14336, 2), M.DTYPE_BF16); w.random(0)
sp = ctx.stream; st = torch.cuda.ExternalStream(sp)
with torch.cuda.stream(st):
    xs = torch.randn((4, 512, 4096), device="cuda"); xo = torch.empty((512, 4096), device="cuda")
    ids = torch.zeros((512, 2), dtype=torch.int32, device="cuda"); g = torch.zeros((512, 2), device="cuda")
torch.cuda.synchronize()
for i in range(4): w.layer_forward(0, xs[i], xo, ids, g, stream=sp)
torch.cuda.synchronize()
PY
for f in 1 0; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_pf$f.csv python /tmp/pf1.py $f > /dev/null 2>&1
python - $f <<'PY'
import csv, sys, collections
f = sys.argv[1]
rows = list(csv.DictReader(open(f"gpurun_out/ncu_pf{f}.csv")))
agg = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        agg[r["Kernel Name"][:60]].append(float(r["Metric Value"].replace(",", "")))
print("fused", f)
for k, v in agg.items(): print(f"  {k:60s} n={len(v)} mean={sum(v)/len(v)/1e3:.1f} us")
PY
done
