#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for v in 256 128 64 0; do
  SATTN_L2_PROMO=$v timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream > $OUT/b_l2$v.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_l2$v.json'));print('promo $v', d['value'], d['roofline']['per_call_ms'])"
done
