#!/bin/bash
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
for o in 0 1 2; do SATTN_FUSED_ORDER=$o timeout 300 python scripts/tc_trace_fused.py > $OUT/fused_o$o.txt 2>&1; done
SATTN_SA_BWD=split timeout 300 python scripts/tc_trace_fused.py > $OUT/split.txt 2>&1
tail -n 4 $OUT/*.txt
