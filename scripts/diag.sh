#!/bin/bash
# Diagnostics session: TMA ingest microbenchmark + per-phase traces of the tensor-core kernels.
OUT=gpurun_out/${1:-diag}; mkdir -p $OUT
( ./scripts/micro/tma_ingest ) > $OUT/tma_ingest.txt 2>&1
for s in tc_trace tc_cta_trace tc_trace_bwd; do timeout 300 python scripts/$s.py > $OUT/$s.txt 2>&1; done
tail -n 60 $OUT/*.txt
