#!/bin/bash
# full evidence pass: GPU tests, the driver's bench lines (ours, reference),
# the ncu launch list of the headline command, ncu full captures of the hot kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_gputests.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?" >> gpurun_out/${T}_bench_ref.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-config --no-red-trace"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_units -s 40 -c 1 -o gpurun_out/${T}_units_c5 python tools/gpu/time_sweep.py 5 1 > gpurun_out/${T}_ncu_units.log 2>&1; echo "units rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 40 -c 1 -o gpurun_out/${T}_p1_c5 python tools/gpu/time_sweep.py 5 1 > gpurun_out/${T}_ncu_p1.log 2>&1; echo "p1 rc=$?"
for c in 3 4 2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 -o gpurun_out/${T}_sweep_c$c python tools/gpu/time_sweep.py $c 1 > gpurun_out/${T}_ncu_c$c.log 2>&1; echo "c$c rc=$?"
done
bash tools/gpu/run_multirank.sh > gpurun_out/${T}_multirank.log 2>&1; echo "multirank done"
