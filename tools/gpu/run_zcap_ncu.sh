#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
MSURF_ZCAP_DEPTH=2 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/zd_launches.csv python tools/gpu/time_sweep.py 5 1 > gpurun_out/zd_ncu.log 2>&1
MSURF_ZCAP_DEPTH=2 ncu --set full --clock-control none --import-source on -k regex:sweep_units -s 60 -c 1 -o gpurun_out/zd_units python tools/gpu/time_sweep.py 5 1 > gpurun_out/zd_full.log 2>&1
MSURF_ZCAP_DEPTH=2 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 60 -c 1 -o gpurun_out/zd_p1 python tools/gpu/time_sweep.py 5 1 > gpurun_out/zd_full2.log 2>&1
