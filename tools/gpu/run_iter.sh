# one optimisation iteration: GPU tests (parity gate) + quick bench config 2 (+ optional configs)
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-2}; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/iter_c$c.json 2> gpurun_out/iter_c$c.err; echo bench rc=$?
python - $c <<'PY'
import json,sys
c=sys.argv[1]
d=json.loads(open(f'gpurun_out/iter_c{c}.json').read().strip().splitlines()[-1])
r=d['roofline']; print('RESULT config', c, 'ms/step %.3f sweep_ms %.3f frac %.3f evald %d atomics %d e2e_ms %.3f value %.3g e2e %.3g clocks %s' % (d['ms_per_step'], r['sweep_ms'], r['frac'], r['points_evaluated'], r['atomics'], d['e2e']['ms_per_step'], d['value'], d['e2e']['value'], d['clocks']))
PY
tail -3 gpurun_out/iter_c$c.err
done
