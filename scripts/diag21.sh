#!/bin/bash
timeout 1300 python -m pytest tests -m gpu -q -x --durations=10 2>&1 | tail -16
timeout 300 python scripts/band_time.py
