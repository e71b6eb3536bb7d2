#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the SA, LLSA and stack/stream scripts
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  for sc in sanitize_band sanitize_llsa sanitize_misc; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/$sc.py > $OUT/$tool-$sc.log 2>&1
    echo "$tool $sc rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/$tool-$sc.log | tail -1)"
  done
done
