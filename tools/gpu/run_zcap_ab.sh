#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/zab_tests.log
for c in 5 2; do timeout 300 python tools/gpu/time_sweep.py $c 5 >> gpurun_out/zab.txt 2>&1; done
MSURF_ZCAP_DEPTH=2 timeout 300 python tools/gpu/time_sweep.py 5 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ depth 2" >> gpurun_out/zab.txt
