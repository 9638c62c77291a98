#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_small.py (every path).
O=${1:-gpurun_out/sanitize}; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_small.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/summary.txt
  tail -3 $O/$tool.log
done
