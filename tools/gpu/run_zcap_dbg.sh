#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
MSURF_ZCAP=0 python tools/gpu/time_sweep.py 5 3 > gpurun_out/zd_off.txt 2>&1
MSURF_ZCAP=1 python tools/gpu/time_sweep.py 5 3 > gpurun_out/zd_on.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/zd_launches.csv python tools/gpu/time_sweep.py 5 1 > gpurun_out/zd_ncu.log 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tile_list_path_equals_per_job_path" > gpurun_out/zd_test.log 2>&1
