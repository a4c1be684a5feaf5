#!/bin/bash
# launch lists (C2q1, C5) + ncu source profile of the TSQR block kernel and the QRCP kernel
mkdir -p gpurun_out
for CFG in C2q1 C5; do
  S=3; [ $CFG = C5 ] && S=1
  CMD="python bench.py --config $CFG --steps $S --warmup 2 --no-cpu-baseline"
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > /dev/null 2>&1
  echo "== $CFG"; python tools/launches_summary.py gpurun_out/launches_$CFG.csv | head -20
done
timeout -s KILL 120 python tools/prof_qr.py > /dev/null 2>&1
for K in k_qr_blocked k_qrcp_reg; do
  timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K -f python tools/prof_qr.py > /dev/null 2>&1
  echo "$K rc=$?"
done
