#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_corutv.py tests/test_gpu_approx.py -q -x --timeout 300 > gpurun_out/t_k.log 2>&1
grep -E "^E |FAILED|passed|failed" gpurun_out/t_k.log | head -20
CORU_GEMM_TILE_SPLIT_CAP=0 timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_corutv.py tests/test_gpu_approx.py -q -x --timeout 300 2>&1 | tail -3
