for nt in 1 4 1 4 8; do
  MSURF_NATIVE_THREADS=$nt python bench.py --config 3 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/nt.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/nt.json').read().strip().splitlines()[-1]); print('NT $nt e2e', round(d['e2e']['ms_per_step'],3), d['e2e']['steps_ms'])"
done
