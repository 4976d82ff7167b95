# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_workload.py
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_workload.py > gpurun_out/san_$t.txt 2>&1; echo "rc=$?" >> gpurun_out/san_$t.txt
  echo "$t: $(grep -h 'SUMMARY' gpurun_out/san_$t.txt | tail -1) $(tail -1 gpurun_out/san_$t.txt)"
done
