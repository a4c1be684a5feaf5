#!/bin/bash
# launch lists of the wide configs (one decomposition each after one warm-up)
mkdir -p gpurun_out
for CFG in C3 C4 C5; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > /dev/null 2>&1
  echo "== $CFG"; python tools/launches_summary.py gpurun_out/launches_$CFG.csv | head -12
done
