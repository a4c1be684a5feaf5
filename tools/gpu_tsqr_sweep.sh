#!/bin/bash
mkdir -p gpurun_out
for t in default 512 1024 2000 4001; do
  if [ $t = default ]; then unset CORU_TSQR_TARGET; else export CORU_TSQR_TARGET=$t; fi
  timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ts_$t.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ts_$t.json'));print('C2q1 target $t', round(d['ms_per_step'],4))"
done
