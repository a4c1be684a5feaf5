#!/bin/bash
mkdir -p gpurun_out
for v in 0 1; do
  CORU_TN_SMALL=$v timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tn_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tn_$v.json'));print('C2q1 tn $v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1))"
  CORU_TN_SMALL=$v timeout -s KILL 300 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tn1_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tn1_$v.json'));print('C1 tn $v', round(d['ms_per_step'],4))"
  CORU_TN_SMALL=$v timeout -s KILL 300 python bench.py --config C2q1 --variant approx --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tn2_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tn2_$v.json'));print('C2q1 approx tn $v', round(d['ms_per_step'],4))"
done
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
grep -E "^E |FAILED|passed|failed" gpurun_out/t_gpu.log | head -12
