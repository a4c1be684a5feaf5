#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench (plain), launch list (ncu, timing only), ncu --set full
# of the A-pass GEMM. Every step bounded so a hung kernel cannot eat the slot.
mkdir -p gpurun_out
CFG=${CFG:-C2q1}
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/ncu_launches.log
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_f64 -s 7 -c 7 -o gpurun_out/prof_gemm_$CFG -f $CMD > gpurun_out/prof_gemm_ncu_$CFG.log 2>&1; echo "full rc=$?" >> gpurun_out/prof_gemm_ncu_$CFG.log
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json; tail -2 gpurun_out/ncu_launches.log gpurun_out/prof_gemm_ncu_$CFG.log
