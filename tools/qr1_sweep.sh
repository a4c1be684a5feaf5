for cfg in C2q1 C2q2 C1; do
for E in late early; do
  if [ $E = early ]; then export CORU_QR1_EARLY=1; else unset CORU_QR1_EARLY; fi
  timeout -s KILL 200 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/q1_$E.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/q1_$E.json')); r=d['roofline']; print('$cfg $E', 'ms/step %.3f' % d['ms_per_step'], 'apass avg %.1f us frac %.3f' % (r['avg_launch_ms']*1e3, r['frac']))"
done; done
