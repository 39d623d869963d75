# run_variants3.sh: bench sweep time per variant library (VARIANTS, CONFIGS env)
for cfg in ${CONFIGS:-3}; do
  for v in ${VARIANTS:-base}; do
    MSURF_LIB=build_variants/libmsurf_$v.so timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v3_${v}_c$cfg.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/v3_${v}_c$cfg.json').read().strip().splitlines()[-1]); print('RESULT $v config $cfg sweep_ms %.4f step %.4f e2e %.4f' % (d['roofline']['sweep_ms'], d['ms_per_step'], d['e2e']['ms_per_step']))" || tail -5 gpurun_out/v3_${v}_c$cfg.json
  done
done
