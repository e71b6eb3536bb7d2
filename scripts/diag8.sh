#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for pf in 0 3 6 10; do
  SATTN_FWD_PF=$pf timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream > $OUT/b_pf$pf.json 2>&1
  python -c "import json;d=json.load(open('$OUT/b_pf$pf.json'));print('pf $pf', d['roofline']['per_call_ms'])"
done
