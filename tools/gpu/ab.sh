python tools/ab_stack.py --layers 4 --iters 20 > gpurun_out/ab4.json 2>&1
python tools/ab_stack.py --layers 32 --scale 0.1 --rounds 5 > gpurun_out/ab32.json 2>&1
cat gpurun_out/ab4.json gpurun_out/ab32.json
