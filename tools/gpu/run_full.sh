# full default bench + reference arm + launch list + full ncu capture of the sweep (tag = $1)
set -x
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
tail -c 400 gpurun_out/bench_${TAG}.json
python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo ref rc=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_${TAG}.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo launches rc=$?
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo full rc=$?
