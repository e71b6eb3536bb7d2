#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
timeout 300 python scripts/tc_trace_bwd.py > $OUT/trace_bwd.txt 2>&1
timeout 300 python scripts/tc_trace_fused.py > $OUT/split.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
[ -n "$BENCH" ] && timeout 600 python bench.py --no-e2e --no-llsa --no-cpu --no-stream > $OUT/bench.json 2>&1
tail -n 14 $OUT/*.txt; tail -c 1500 $OUT/bench.json
