#!/bin/bash
timeout 300 python scripts/band_time.py
timeout 300 python scripts/band_time.py 32 16
timeout 300 python scripts/band_time.py 16 8
