# like run_variants.sh but base runs with MSURF_ONE_JOB_MAX=0 (old batched path)
for cfg in ${CONFIGS:-2}; do
  MSURF_ONE_JOB_MAX=0 MSURF_LIB=build_variants/libmsurf_base.so python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v2_base_c$cfg.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/v2_base_c$cfg.json').read().strip().splitlines()[-1]); print('RESULT base config $cfg sweep_ms %.4f step %.4f' % (d['roofline']['sweep_ms'], d['ms_per_step']))"
  for v in build_variants/libmsurf_one*.so; do
    MSURF_LIB=$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v2_c$cfg.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/v2_c$cfg.json').read().strip().splitlines()[-1]); print('RESULT $v config $cfg sweep_ms %.4f step %.4f' % (d['roofline']['sweep_ms'], d['ms_per_step']))" || tail -5 gpurun_out/v2_c$cfg.json
  done
done
