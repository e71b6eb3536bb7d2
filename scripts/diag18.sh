#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -15
timeout 120 python scripts/band_time.py
timeout 120 python scripts/band_time.py 32 16
