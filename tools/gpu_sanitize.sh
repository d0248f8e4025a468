D=gpurun_out/sanitize; mkdir -p $D
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 --log-file $D/$tool.log python tools/sanitize_cases.py small > $D/$tool.out 2>&1
  echo "$tool rc=$?" >> $D/summary.txt
done
timeout 1200 $CS --tool memcheck --print-limit 50 --log-file $D/memcheck_full.log python tools/sanitize_cases.py full > $D/memcheck_full.out 2>&1
echo "memcheck_full rc=$?" >> $D/summary.txt
