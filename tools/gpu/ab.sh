python tools/ab_stack.py --layers 4 --iters 20 --configs 1,2:0,2:1 > gpurun_out/ab4.json 2>&1
python tools/ab_stack.py --layers 32 --scale 0.1 --rounds 3 --configs 1,2:0,2:1:8,2:1:16,2:1:32 > gpurun_out/ab32.json 2>&1
python tools/trace_stack.py --reps 2 --out gpurun_out/trace_bal.json > /dev/null 2>&1
grep "tok_s\|determ\|ids_eq\|normw" gpurun_out/ab4.json gpurun_out/ab32.json; tail -3 gpurun_out/ab32.json
