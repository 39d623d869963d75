set -x
for cfg in ${CFGS:-4}; do
for mb in ${MBS:-12 24 32 48}; do
  MSURF_L2_TILE_MB=$mb python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/l2_${cfg}_$mb.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/l2_${cfg}_$mb.json').read().strip().splitlines()[-1]); print('RESULT cfg $cfg tile_mb $mb sweep_ms', d['roofline']['sweep_ms'], 'step', d['ms_per_step'])"
done; done
