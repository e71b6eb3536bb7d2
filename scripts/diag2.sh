#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
timeout 300 python scripts/tc_trace_fused.py > $OUT/fused.txt 2>&1
[ -n "$SPLIT" ] && SATTN_SA_BWD=split timeout 300 python scripts/tc_trace_fused.py > $OUT/split.txt 2>&1
[ -n "$TESTS" ] && timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1
tail -n 40 $OUT/*.txt
