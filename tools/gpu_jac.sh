#!/bin/bash
for v in 0 1 2; do CORU_JACOBI_VARIANT=$v timeout -s KILL 120 python tools/jacobi_ab.py 2>&1 | grep variant; done
for v in 0 1 2; do
  CORU_JACOBI_VARIANT=$v timeout -s KILL 300 python bench_rpca.py --no-cpu-baseline > gpurun_out/br_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/br_$v.json'));print('rpca variant $v', round(d['ms_per_step'],2))"
done
for v in 1 2; do CORU_JACOBI_VARIANT=$v timeout -s KILL 600 python -m pytest tests/test_gpu_baselines.py tests/test_gpu_approx.py tests/test_gpu_rpca.py -q -x --timeout 300 2>&1 | tail -1; done
