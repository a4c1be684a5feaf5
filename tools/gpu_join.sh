#!/bin/bash
for v in late early; do
  if [ $v = early ]; then export CORU_EARLY_JOIN=1; fi
  timeout -s KILL 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/j_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/j_$v.json'));print('C2q1 $v', round(d['ms_per_step'],4))"
  timeout -s KILL 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/j3_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/j3_$v.json'));print('C3 $v', round(d['ms_per_step'],3))"
done
unset CORU_EARLY_JOIN
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
