# compute-sanitizer over tools/sanitize_probe.py (memcheck, racecheck,
# synccheck); summaries land in gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_probe.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_$tool.txt
  tail -3 gpurun_out/sanitize_$tool.txt
done
