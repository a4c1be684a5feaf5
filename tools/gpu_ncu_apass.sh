#!/bin/bash
# ncu --set full of the A-pass kernels of C3, C4, C5 (one decomposition's first passes), one GPU.
mkdir -p gpurun_out
for cfg in C3 C4; do
  timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_f64 -s 0 -c 4 \
    -o gpurun_out/prof_apass_$cfg -f python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_apass_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_apass_tf32x3 -s 0 -c 2 \
  -o gpurun_out/prof_apass_C5 -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_apass_C5.log 2>&1
echo "C5 rc=$?"
