#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for o in 0 1 2; do
  SATTN_MMA_ORDER=$o timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream --no-hour > $OUT/b_o$o.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_o$o.json'));print('order $o', d['value'], d['roofline']['per_call_ms'])"
done
