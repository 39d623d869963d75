#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for d in 1 2 3 4; do for w in 0 1; do
MSURF_ZCAP_DEPTH=$d MSURF_ZCAP_WIDE=$w timeout 300 python tools/gpu/time_sweep.py 5 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ c5 depth=$d wide=$w" >> gpurun_out/zab.txt
done; done
for d in 2 4 8; do
MSURF_ZCAP_MIN_JOBS=1 MSURF_ZCAP_DEPTH=$d timeout 300 python tools/gpu/time_sweep.py 2 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ c2 depth=$d" >> gpurun_out/zab.txt
done
MSURF_ZCAP=0 timeout 300 python tools/gpu/time_sweep.py 5 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ c5 nocap" >> gpurun_out/zab.txt
