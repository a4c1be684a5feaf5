#!/bin/bash
# tcgen05 fp32 A-pass: kernel parity tests, fp32 decomposition tests, C5 bench (bounded).
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "tensor_core" --timeout 120 > gpurun_out/t_tc.log 2>&1; echo "rc=$?" >> gpurun_out/t_tc.log
tail -30 gpurun_out/t_tc.log
if grep -q "passed" gpurun_out/t_tc.log && ! grep -q "failed\|error" gpurun_out/t_tc.log; then
  timeout -s KILL 600 python -m pytest tests/test_gpu_corutv.py tests/test_gpu_fullsize.py -q -x -k "f32 or C5 or fp32" --timeout 300 > gpurun_out/t_f32.log 2>&1; echo "rc=$?" >> gpurun_out/t_f32.log
  tail -5 gpurun_out/t_f32.log
  timeout -s KILL 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
fi
