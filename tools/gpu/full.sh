free -g | head -2 > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -25 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench.err; cat gpurun_out/host_mem.txt
