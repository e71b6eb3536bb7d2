#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "k2_variants" 2>&1 | tail -3
for v in old rm64 m64; do
  SATTN_K2=$v timeout 300 python bench.py --steps 10 --no-e2e --no-llsa --no-cpu --no-stream --no-hour --no-encoder > gpurun_out/k2_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/k2_$v.json'));print('K2 $v', d['value'], d['roofline']['per_call_ms'])"
done
