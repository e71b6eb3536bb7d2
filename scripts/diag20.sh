#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -5
timeout 300 python scripts/band_time.py 32 16
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu --no-stream --no-hour --no-encoder --no-llsa > gpurun_out/band_bench.json 2>gpurun_out/band_bench.err
python -c "import json;d=json.load(open('gpurun_out/band_bench.json'));print(d['value'], d['roofline']['per_call_ms'], json.dumps(d['band']))"
