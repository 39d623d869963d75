#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suite_gpu.py -m gpu -x -q > gpurun_out/refsuite.log 2>&1
for c in 3 4 2 5 1; do
timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-per-config --no-cpu-baseline > gpurun_out/replay_c$c.json 2> gpurun_out/replay_c$c.err
done
