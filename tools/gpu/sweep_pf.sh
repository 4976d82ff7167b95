# grouped prefill kernel tail knobs: layer-time sweep + per-tile traces at K splits 2 / 4 / 8
timeout 900 python tools/sweep_prefill_splits.py --rounds 3 --cfgs "${1:-2:3,4:3,8:3,8:3:2,8:8:8,2:3:0:2,2:3:0:4,4:3:0:4,2:8:1}" > gpurun_out/sweep_pf.json 2>&1
cat gpurun_out/sweep_pf.json
for S in 2 4 8; do echo "== prefill_splits=$S"; timeout 300 python tools/trace_prefill.py --reps 1 --opt prefill_splits=$S 2>&1 | tail -4; done
