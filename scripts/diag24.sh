#!/bin/bash
for i in 1 2; do
SATTN_LIB=$PWD/libsattn_oldwait.so timeout 300 python scripts/band_time.py
timeout 300 python scripts/band_time.py
done
