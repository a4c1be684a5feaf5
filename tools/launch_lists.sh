#!/bin/bash
# ncu launch lists (timing only) of one decomposition per config + the NCCL world-1 plumbing test
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_sharded.py -q -x -k nccl --timeout 200 2>&1 | tail -3
for cfg in C3 C4 C5; do
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "== $cfg rc=$?"; python tools/launches_summary.py gpurun_out/launches_$cfg.csv | head -14
done
