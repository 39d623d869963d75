#!/bin/bash
# A/B of engine env knobs on bench lines: ENVS="base|K=V|..." CONFIGS="5" TAG=x bash tools/gpu/run_env_ab.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-envab}
IFS='|' read -ra KV <<< "${ENVS:-base}"
for c in ${CONFIGS:-5}; do
  n=0
  for kv in "${KV[@]}"; do
    if [ "$kv" = base ]; then E=""; else E="$kv"; fi
    echo "$kv" > gpurun_out/${T}_c${c}_$n.env
    env $E timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-per-config --no-cpu-baseline --no-red-trace > gpurun_out/${T}_c${c}_$n.json 2> gpurun_out/${T}_c${c}_$n.err
    n=$((n+1))
  done
done
