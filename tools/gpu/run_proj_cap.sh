#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python tools/gpu/project_strips.py --configs 5 2 4 > gpurun_out/project_r2c.jsonl 2> gpurun_out/project_r2c.err
for c in 2 5; do timeout 300 python tools/gpu/time_sweep.py $c 5 >> gpurun_out/zab2.txt 2>&1; done
