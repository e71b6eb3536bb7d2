#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_band.py -q -x 2>&1 | tail -1
timeout 300 python scripts/band_time.py
timeout 300 python scripts/band_time.py
