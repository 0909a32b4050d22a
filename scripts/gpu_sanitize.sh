#!/bin/bash
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  for m in cnn speech lstm logreg; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_round.py $m > gpurun_out/san_${tool}_${m}.log 2>&1
    echo "$tool $m rc=$?" >> gpurun_out/san_summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok " gpurun_out/san_${tool}_${m}.log >> gpurun_out/san_summary.txt
  done
done
