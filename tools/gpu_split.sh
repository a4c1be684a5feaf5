#!/bin/bash
mkdir -p gpurun_out
for cap in 0 8 16 32; do
  CORU_GEMM_TILE_SPLIT_CAP=$cap timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/split_$cap.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/split_$cap.json'));print('cap $cap', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), 'apass', round(d['roofline']['achieved'],2))"
done
for cap in 0 16; do
  CORU_GEMM_TILE_SPLIT_CAP=$cap timeout -s KILL 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/split_c4_$cap.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/split_c4_$cap.json'));print('C4 cap $cap', round(d['ms_per_step'],3))"
  CORU_GEMM_TILE_SPLIT_CAP=$cap timeout -s KILL 300 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/split_c1_$cap.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/split_c1_$cap.json'));print('C1 cap $cap', round(d['ms_per_step'],4))"
done
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_corutv.py tests/test_gpu_approx.py -q -x --timeout 300 2>&1 | tail -2
