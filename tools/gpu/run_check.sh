#!/bin/bash
# correctness (full GPU suite) + quick per-config timings
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
for c in ${CONFIGS:-3 4 2 5 1}; do
timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-per-config --no-cpu-baseline > gpurun_out/${T}_c$c.json 2> gpurun_out/${T}_c$c.err
done
