#!/bin/bash
for nw in 16 32 8; do
  CORU_QRCP_NW=$nw timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/nw_$nw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/nw_$nw.json'));print('C2q1 nw $nw', round(d['ms_per_step'],4))"
done
CORU_QRCP_NW=32 timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_corutv.py -q -x --timeout 300 -k "qrcp or reference_cases or config" 2>&1 | tail -1
CORU_QRCP_NW=8 timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_corutv.py -q -x --timeout 300 -k "qrcp or reference_cases or config" 2>&1 | tail -1
