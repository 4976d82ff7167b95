for f in 1 0; do echo "== prefill_fused=$f"; timeout 300 python tools/trace_prefill.py --reps 2 --opt prefill_fused=$f 2>&1 | tail -5; done
