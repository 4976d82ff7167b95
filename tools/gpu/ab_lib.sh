#!/bin/bash
# Interleaved A/B of two library builds through bench.py (A = $MOE_AB_LIB_A,
# default paper_2402_07033_b200/_build_ab/libmoe_b200.so; B = the in-tree build).
# usage: bash tools/gpu/ab_lib.sh "<bench args>" [rounds]
ARGS=${1:-"--config layer --steps 1000 --warmup 20"}
A=${MOE_AB_LIB_A:-$PWD/paper_2402_07033_b200/_build_ab/libmoe_b200.so}
for r in $(seq 1 ${2:-3}); do
  for v in A B; do
    if [ $v = A ]; then export MOE_B200_LIB=$A; else unset MOE_B200_LIB; fi
    timeout 300 python bench.py --no-extras --no-cpu-baseline $ARGS > gpurun_out/ab_${v}_r${r}.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${v}_r${r}.json')); print('$v r$r', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_us'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
