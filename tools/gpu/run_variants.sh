# sweep timing for each libmsurf variant in build_variants/ (optionally pytest first: RUN_TESTS=1)
set -x
if [ "${RUN_TESTS:-0}" = "1" ]; then
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
fi
for v in build_variants/libmsurf_*.so; do
  for cfg in ${CONFIGS:-2}; do
  MSURF_LIB=$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_$(basename $v .so)_c$cfg.json 2>&1
  python - "$v" "$cfg" <<'PY'
import json,sys
v=sys.argv[1]; c=sys.argv[2]
try:
    d=json.loads(open('gpurun_out/var_'+v.split('/')[-1][:-3]+'_c'+c+'.json').read().strip().splitlines()[-1])
    r=d['roofline']; print('RESULT', v, 'config', c, 'ms/step %.3f sweep_ms %.3f frac %.3f atomics %d e2e %.3f' % (d['ms_per_step'], r['sweep_ms'], r['frac'], r['atomics'], d['e2e']['ms_per_step']))
except Exception as e: print('RESULT', v, 'ERR', e)
PY
  done
done
