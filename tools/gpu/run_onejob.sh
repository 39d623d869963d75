# per-job (by-value) vs batched sweep launches for launch groups of many surfaces
for v in 32 0; do
  echo "=== MSURF_ONE_JOB_MAX=$v"
  MSURF_ONE_JOB_MAX=$v python tools/gpu/e2e_timeline3.py 2>&1 | head -40
  for c in 4 5 3; do
    MSURF_ONE_JOB_MAX=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config $c ms', round(d['ms_per_step'],3), 'sweep', round(d['roofline']['sweep_ms'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
  done
done
