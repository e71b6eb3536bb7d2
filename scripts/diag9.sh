#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for sl in 0 20 100 400; do
  SATTN_MMA_SLEEP=$sl timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream > $OUT/b_sl$sl.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_sl$sl.json'));print('sleep $sl', d['value'], d['roofline']['per_call_ms'])"
done
