#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for m in 0 1 3; do
  SATTN_POLY=$m timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream --no-hour > $OUT/b_p$m.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_p$m.json'));print('poly $m', d['value'], d['roofline']['per_call_ms'])"
done
SATTN_POLY=1 timeout 600 python -m pytest tests -m gpu -x -q -k "sa_bf16 or full" 2>&1 | tail -2
