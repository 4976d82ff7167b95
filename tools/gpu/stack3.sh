# decode_stack3 A/B: bit-equality tests, A/B timing vs stack 2, phase trace.
timeout 600 python -m pytest tests/test_gpu_stack3.py -q -x > gpurun_out/pytest_stack3.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_stack3.txt
timeout 600 python tools/ab_stack.py --layers 32 --scale 0.1 --rounds 5 --iters 30 --kernels 2,3 --configs 2,3,2,3 > gpurun_out/ab32_k3.json 2>&1
timeout 300 python tools/trace_stack3.py --reps 2 --out gpurun_out/trace_k3.json > gpurun_out/trace_k3.txt 2>&1
tail -3 gpurun_out/pytest_stack3.txt; cat gpurun_out/ab32_k3.json; cat gpurun_out/trace_k3.txt
