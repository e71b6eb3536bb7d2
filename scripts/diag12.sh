#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "coop or ring" 2>&1 | tail -3
for v in old coop; do
  SATTN_K2=$v timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream --no-hour > $OUT/b_$v.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_$v.json'));print('K2 $v', d['value'], d['roofline']['per_call_ms'])"
done
SATTN_K2=coop timeout 300 python scripts/tc_trace_bwd.py | tail -11
