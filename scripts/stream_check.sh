#!/bin/bash
# incremental-step kernels: parity tests + the bench's stream timing only
OUT=gpurun_out/${1:-stream}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stack_stream.py -q -x -k "stream" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 600 python - > $OUT/stream.json 2>$OUT/stream.err <<'PY'
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2302_13451_b200 as s
print(json.dumps(bench.run_stream(s, torch.device("cuda", 0))))
PY
cat $OUT/stream.json; tail -3 $OUT/stream.err
