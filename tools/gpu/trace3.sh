M=${1:-3}
timeout 300 python tools/trace_stack3.py --reps 2 --kernel $M --out gpurun_out/trace_k3.json > gpurun_out/trace_k3.txt 2>&1
cat gpurun_out/trace_k3.txt
