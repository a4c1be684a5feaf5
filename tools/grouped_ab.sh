#!/bin/bash
# A/B of grouped stream-K (CORU_GEMM_GROUPED) on the multi-n-tile configs + kernel tests
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 300 -k "gemm" 2>&1 | tail -2
for G in 1 0; do
  export CORU_GEMM_GROUPED=$G
  for cfg in C3 C4; do
    timeout -s KILL 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g_${cfg}_$G.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/g_${cfg}_$G.json')); r=d['roofline']; print('$cfg grouped=$G', 'ms/step %.2f' % d['ms_per_step'], 'apass %.1f us frac %.3f' % (r['avg_launch_ms']*1e3, r['frac']))"
  done
done
export CORU_GEMM_GROUPED=1
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_gemm_f64 -s 0 -c 4 --csv python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | cut -d, -f5,13-16 | head -8
