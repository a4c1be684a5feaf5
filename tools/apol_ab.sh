#!/bin/bash
for P in 0 1 2; do
  export CORU_GEMM_APOL=$P
  for cfg in C3 C4; do
    timeout -s KILL 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p_${cfg}_$P.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/p_${cfg}_$P.json')); r=d['roofline']; print('$cfg apol=$P', 'ms/step %.2f' % d['ms_per_step'], 'apass %.1f us frac %.3f' % (r['avg_launch_ms']*1e3, r['frac']))"
  done
  timeout -s KILL 600 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:k_gemm_f64 -s 0 -c 4 --csv python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/p_ncu_$P.csv
  python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/p_ncu_$P.csv")) if len(r) > 14 and r[12] == "dram__bytes_read.sum"]
print("C4 apol=$P dram read per launch (x A):", [round(float(r[14].replace(",",""))*{"Gbyte":1e9,"Mbyte":1e6}.get(r[13],1)/8.59e9, 2) for r in rows])
PY
done
