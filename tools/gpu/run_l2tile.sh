set -x
for mb in 6 12 24 48 96; do
  MSURF_L2_TILE_MB=$mb python bench.py --config ${CFG:-4} --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/l2_$mb.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/l2_$mb.json').read().strip().splitlines()[-1]); print('RESULT tile_mb $mb sweep_ms', d['roofline']['sweep_ms'], 'step', d['ms_per_step'])"
done
