#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x -k "k2_variants or sa_bf16 or stored_band or full" 2>&1 | tail -1
timeout 300 python scripts/band_time.py 32 32
SATTN_K2=coop timeout 300 python scripts/band_time.py 32 8
