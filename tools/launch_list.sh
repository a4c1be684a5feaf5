#!/bin/bash
# Per-launch device times of one bench run (ncu, cold-cache/serialised: compare SHARES).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu.log
