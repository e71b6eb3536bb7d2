#!/bin/bash
# cold, serialised per-kernel durations of the stored-band backward (ncu launch list; shares only)
OUT=gpurun_out/${1:-bk}; mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sa_bwd" --csv --log-file $OUT/k.csv python scripts/bwd_chunk.py > /dev/null 2>&1
python - "$OUT/k.csv" <<'PY'
import csv, collections, sys
d = collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 14 and r[-3] == "gpu__time_duration.sum":
        d[r[4].split("(")[0]].append(float(r[-1].replace(",", "")))
for k, v in d.items():
    v = sorted(v); print(k, len(v), "median us", v[len(v) // 2] / 1e3)
PY
