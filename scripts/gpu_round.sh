#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list and a full capture of the top kernels.
# usage: bash scripts/gpu_round.sh [tag]   (outputs land in gpurun_out/<tag>/)
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvidia-smi.csv 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 900 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-llsa --no-cpu --no-stream --no-hour --no-encoder --no-alt $NCU_BENCH_ARGS > $OUT/ncu_launch_run.log 2>&1
  echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KREGEX:-sa_.*_tc|ffma}" -s ${NCU_SKIP:-47} -c ${NCU_COUNT:-3} \
      -o $OUT/prof_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-llsa --no-cpu --no-stream --no-hour --no-encoder --no-alt $NCU_BENCH_ARGS > $OUT/ncu_full_run.log 2>&1
  echo "ncu full rc=$?"
fi
ls -la $OUT
