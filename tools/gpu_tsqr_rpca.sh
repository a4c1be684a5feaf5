#!/bin/bash
for t in default 1024 700 2000; do
  if [ $t = default ]; then unset CORU_TSQR_TARGET; else export CORU_TSQR_TARGET=$t; fi
  timeout -s KILL 300 python bench_rpca.py --no-cpu-baseline > gpurun_out/tr_$t.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/tr_$t.json'));print('rpca target $t', round(d['ms_per_step'],2), d['config']['iterations'])"
done
