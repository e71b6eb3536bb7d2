#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
SATTN_FUSED_PREFETCH=1 timeout 300 python scripts/tc_trace_fused.py > $OUT/fused_pf1.txt 2>&1
SATTN_FUSED_PREFETCH=0 timeout 300 python scripts/tc_trace_fused.py > $OUT/fused_pf0.txt 2>&1
tail -n 16 $OUT/*.txt
