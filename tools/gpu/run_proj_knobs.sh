#!/bin/bash
# config-5 strip projection under capped-launch knobs (engine.py MSURF_ZCAP_*):
# KNOBS="base|MSURF_ZCAP_DEPTH=2|..." NS="1 2 8" TAG=x bash tools/gpu/run_proj_knobs.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-pk}
IFS='|' read -ra KV <<< "${KNOBS:-base}"
for kv in "${KV[@]}"; do
  if [ "$kv" = base ]; then E=""; else E="$kv"; fi
  echo "== $kv" >> gpurun_out/${T}.jsonl
  env $E timeout 600 python tools/gpu/project_strips.py --configs ${CONFIGS:-5} --ns ${NS:-1 2 8} --steps 3 >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
done
