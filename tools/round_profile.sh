#!/bin/bash
# One GPU call's worth of round evidence (run under gpurun from the repo root):
# tests, smoke, bench lines (decode stack + prefill), the ncu launch list of
# the bench command and one `ncu --set full` capture per top kernel.
# Outputs under gpurun_out/$TAG/.
TAG=${1:-round}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_stack32.json 2> $O/bench_stack32.err
timeout 300 python bench.py --config prefill512 --no-cpu-baseline > $O/bench_prefill512.json 2> $O/bench_prefill512.err
timeout 300 python bench.py --config layer --no-cpu-baseline --steps 200 > $O/bench_layer.json 2> $O/bench_layer.err
# launch list (cold-cache, serialised: shares, not absolutes)
# (our kernels only: -k skips the one-time random-init launches)
K='regex:decode|reduce|router|permute|prefill|combine|gather|add_kernel'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 400 --csv \
  --log-file $O/launches_stack32.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 200 --csv \
  --log-file $O/launches_prefill512.csv python bench.py --config prefill512 --steps 10 --warmup 3 > /dev/null 2>&1
# full captures of the top kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_stack -s 3 -c 1 \
  -o $O/stack_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_stack -s 3 -c 1 \
  -o $O/layer_full python tools/prof_layer_stack.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefill_grouped|router_topk|combine" -s 6 -c 3 \
  -o $O/prefill_full python tools/prof_prefill.py --iters 3 --no-prof > /dev/null 2>&1
ls -la $O
