#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_rpca.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -8
timeout -s KILL 300 python tools/rpca_check.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print(d['name'], d.get('it'), d.get('rank'), '%.1e %.1e %.1e' % (d['l_rel'], d['s_rel'], d['zeta_rel']))
    except Exception as e: print(l[:200])"
timeout -s KILL 600 python bench_rpca.py > gpurun_out/bench_rpca.json 2> gpurun_out/bench_rpca.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_rpca.json')); r=d['roofline_update']
print('ms/solve', round(d['ms_per_step'],2), 'upd ms', round(r['avg_launch_ms'],3), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2))"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_rpca_lift_update -c 1 -o gpurun_out/rpca_upd python bench_rpca.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_rpca.log 2>&1; echo "ncu rc=$?"
