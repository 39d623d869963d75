#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for d in 1 2 3; do
MSURF_ZCAP_DEPTH=$d timeout 300 python tools/gpu/time_sweep.py 5 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ c5 staged depth=$d" >> gpurun_out/zab.txt
done
MSURF_ZCAP_STAGED=0 MSURF_ZCAP_DEPTH=3 timeout 300 python tools/gpu/time_sweep.py 5 5 >> gpurun_out/zab.txt 2>&1; echo "  ^ c5 unstaged depth=3" >> gpurun_out/zab.txt
MSURF_ZCAP_DEPTH=2 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/zd_launches.csv python tools/gpu/time_sweep.py 5 1 > gpurun_out/zd_ncu.log 2>&1
