# correctness + sweep timing for each libmsurf variant in build_variants/
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
for v in build_variants/libmsurf_*.so; do
  MSURF_LIB=$v python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/var_$(basename $v .so).json 2>&1
  echo $v rc=$?
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open('gpurun_out/var_'+v.split('/')[-1][:-3]+'.json').read().strip().splitlines()[-1])
    r=d['roofline']; print(v, 'ms/step %.3f sweep_ms %.3f frac %.3f atomics %d e2e %.3f' % (d['ms_per_step'], r['sweep_ms'], r['frac'], r['atomics'], d['e2e']['ms_per_step']))
except Exception as e: print(v, 'ERR', e)
PY
done
