#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python scripts/band_time.py
timeout 300 python scripts/band_time.py
timeout 300 python scripts/band_time.py 32 16
