#!/bin/bash
# round-2 evidence: the headline bench line, its ncu launch list, full ncu
# captures of the production sweep kernel for configs 5, 3 and 4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-config"
$CMD > gpurun_out/r02_plain.json 2> gpurun_out/r02_plain.err; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu_launch.log 2>&1; echo launches rc=$?
for c in 5 3 4; do
  python tools/gpu/time_sweep.py $c 3 > gpurun_out/r02_time_c$c.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/r02_sweep_c$c python tools/gpu/time_sweep.py $c 1 > gpurun_out/r02_ncu_full_c$c.log 2>&1
  echo full c$c rc=$?
done
