# usage: bash tools/gpu/run_ncu.sh <tag>
set -x
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_${TAG}.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo launches rc=$?
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo full rc=$?
ls -la gpurun_out
