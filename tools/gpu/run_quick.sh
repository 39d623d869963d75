# correctness + one bench line (no CPU baseline)
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1])
r=d['roofline']; print('ms/step %.3f sweep_ms %.3f frac %.3f evald %d atomics %d e2e_ms %.3f value %.3g e2e %.3g clocks %s' % (d['ms_per_step'], r['sweep_ms'], r['frac'], r['points_evaluated'], r['atomics'], d['e2e']['ms_per_step'], d['value'], d['e2e']['value'], d['clocks']))
PY
tail -5 gpurun_out/bench_quick.err
