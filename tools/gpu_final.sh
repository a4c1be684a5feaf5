#!/bin/bash
# Round-end verification on one B200: full GPU suite, smoke, default bench + reference arm,
# launch list of our kernels, RPCA bench + ncu of its fused update kernel, out-of-core bench.
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
tail -4 gpurun_out/t_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 python bench_rpca.py > gpurun_out/bench_rpca.json 2> gpurun_out/bench_rpca.err; echo "rpca rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rpca_lift_update -c 1 -o gpurun_out/rpca_upd python bench_rpca.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rpca.log 2>&1; echo "ncu rpca rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 3000 --csv --log-file gpurun_out/rpca_launches.csv python bench_rpca.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rpca2.log 2>&1; echo "ncu rpca2 rc=$?"
timeout -s KILL 900 python tools/bench_ooc.py C3 C4 C5 > gpurun_out/bench_ooc.jsonl 2> gpurun_out/bench_ooc.err; echo "ooc rc=$?"
