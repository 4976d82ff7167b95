# bench.py A/B of library configurations, interleaved on one box (no extras, no CPU leg).
# usage: bash tools/gpu/ab_bench.sh "stack_kernel=2 stack_kernel=3,stack3_hold=0" [rounds]
CFGS=${1:-"stack_kernel=2 stack_kernel=3"}
for r in $(seq 1 ${2:-3}); do
  for c in $CFGS; do
    OPTS=$(echo $c | tr ',' '\n' | sed 's/^/--opt /' | tr '\n' ' ')
    tag=$(echo $c | tr ',=' '_-')
    timeout 300 python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline $OPTS > gpurun_out/abb_${tag}_r${r}.json 2>gpurun_out/abb.err
    python -c "import json,sys; d=json.load(open('gpurun_out/abb_${tag}_r${r}.json')); print('$c r$r', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_us'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
