#!/bin/bash
# A/B of a build variant (MSURF_LIB=build_variants/<v>.so) on chosen configs:
# VARIANTS="lp0" CONFIGS="3 4" TAG=x bash tools/gpu/run_ab.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-ab}
for c in ${CONFIGS:-3 4}; do
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then L=""; else L="build_variants/$v.so"; fi
    MSURF_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-per-config --no-cpu-baseline --no-red-trace > gpurun_out/${T}_c${c}_$v.json 2> gpurun_out/${T}_c${c}_$v.err
  done
done
