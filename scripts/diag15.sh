#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "llsa or stack or stream or smoke or full" 2>&1 | tail -2
bash scripts/quick_bench.sh qb16
SATTN_LLSA_NOSKEW=1 bash scripts/quick_bench.sh qb16b
