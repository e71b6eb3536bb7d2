#!/bin/bash
SATTN_FWD_P_LATE=1 timeout 600 python -m pytest tests/test_gpu_band.py -q -x 2>&1 | tail -1
for v in 0 1; do SATTN_FWD_P_LATE=$v timeout 300 python scripts/band_time.py; done
