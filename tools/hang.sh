#!/bin/bash
mkdir -p gpurun_out
for t in "tests/test_gpu_kernels.py -k qrcp" "tests/test_gpu_kernels.py -k tsqr" "tests/test_gpu_kernels.py -k gemm" "tests/test_gpu_corutv.py -k reference_cases" ; do
  echo "== $t" >> gpurun_out/hang.log
  timeout -s KILL 120 python -m pytest $t -m gpu -x -q --timeout 60 --timeout-method=thread >> gpurun_out/hang.log 2>&1
  echo "rc=$?" >> gpurun_out/hang.log
done
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> gpurun_out/hang.log 2>&1
grep -E "==|rc=|passed|failed|Timeout|File" gpurun_out/hang.log | head -60
