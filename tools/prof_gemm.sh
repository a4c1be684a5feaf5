#!/bin/bash
# ncu --set full of one decomposition's 7 GEMM launches (5 A-passes) inside a short bench run
mkdir -p gpurun_out
CFG=${1:-C2q1}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
timeout -s KILL 600 $CMD > gpurun_out/prof_gemm_plain_$CFG.log 2>&1 || { echo plain failed; exit 1; }
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_f64 -s 7 -c 7 -o gpurun_out/prof_gemm_$CFG -f $CMD > gpurun_out/prof_gemm_ncu_$CFG.log 2>&1
echo "$CFG ncu rc=$?"
