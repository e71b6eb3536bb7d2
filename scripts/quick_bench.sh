#!/bin/bash
# quick A/B: SA + LLSA step numbers only
OUT=gpurun_out/${1:-qb}; mkdir -p $OUT
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu --no-stream --no-hour --no-encoder > $OUT/bench.json 2>$OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('SA', d['value'], d['ms_per_step'], d['roofline']['per_call_ms'], 'LLSA', d['llsa']['value'], d['llsa']['ms_per_step'])"
