# bench.py A/B of stack kernels, interleaved on one box (no extras, no CPU leg).
# usage: bash tools/gpu/ab_bench.sh "2 3" [rounds]
CFGS=${1:-"2 3"}
for r in $(seq 1 ${2:-3}); do
  for k in $CFGS; do
    timeout 300 python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline --stack-kernel $k > gpurun_out/abb_${k}_r${r}.json 2>gpurun_out/abb.err
    python -c "import json,sys; d=json.load(open('gpurun_out/abb_${k}_r${r}.json')); print('k$k r$r', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_us'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
