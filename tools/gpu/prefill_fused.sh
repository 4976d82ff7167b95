timeout 900 python -m pytest tests/test_gpu_prefill_fused.py tests/test_gpu_parity.py tests/test_gpu_parity_full.py -q -x -k "fused or prefill or P_ or forward_host or combine or kernel_timing or sparsity or edge" > gpurun_out/pytest_pf.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pf.txt
tail -30 gpurun_out/pytest_pf.txt
timeout 300 python bench.py --config prefill512 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err; tail -2 gpurun_out/bench_pf.err
python -c "import json; d=json.load(open('gpurun_out/bench_pf.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline'])"
