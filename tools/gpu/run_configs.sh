set -x
for c in ${CONFIGS:-3 4 5}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err; echo config $c rc=$?
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f'gpurun_out/cfg{c}.json').read().strip().splitlines()[-1])
    r=d['roofline']; print('RESULT config', c, 'ms/step %.3f sweep_ms %.3f frac %.3f P_eng %d evald %d atomics %d e2e_ms %.3f value %.3g surf/s %.3g' % (d['ms_per_step'], r['sweep_ms'], r['frac'], r['survey_def']['P_eng'], r['points_evaluated'], r['atomics'], d['e2e']['ms_per_step'], d['value'], d['surfaces_per_s']))
except Exception as e: print('RESULT config', c, 'ERR', e)
PY
  tail -3 gpurun_out/cfg$c.err
done
