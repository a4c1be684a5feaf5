timeout -s KILL 600 python -m pytest tests/test_gpu_approx.py tests/test_gpu_baselines.py tests/test_gpu_sharded.py -q -x --timeout 300 2>&1 | tail -3
python tools/pinv_probe.py
for P in 1 0; do
  export CORU_PINV_PRECOND=$P
  for cfg in C2q1 C3; do
    timeout -s KILL 300 python bench.py --config $cfg --variant approx --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pa_${cfg}_$P.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/pa_${cfg}_$P.json')); print('$cfg approx precond=$P ms/step %.3f' % d['ms_per_step'])"
  done
done
