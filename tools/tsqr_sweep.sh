for T in default 1024 1000 700 512 2000; do
  if [ $T = default ]; then unset CORU_TSQR_TARGET; else export CORU_TSQR_TARGET=$T; fi
  timeout -s KILL 200 python bench.py --config C2q1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ts_$T.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ts_$T.json')); print('$T', 'ms/step %.3f' % d['ms_per_step'])"
done
unset CORU_TSQR_TARGET
for T in default 1024 512; do
  if [ $T = default ]; then unset CORU_TSQR_TARGET; else export CORU_TSQR_TARGET=$T; fi
  timeout -s KILL 200 python bench.py --config C2q2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ts2_$T.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ts2_$T.json')); print('C2q2 $T', 'ms/step %.3f' % d['ms_per_step'])"
done
