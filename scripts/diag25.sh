#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in 0 1; do SATTN_FWD_P_LATE=$v timeout 300 python scripts/band_time.py; done
