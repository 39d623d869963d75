# ncu --set full of the sweep kernel for one config: bash tools/gpu/run_ncu_cfg.sh <tag> <config>
set -x
TAG=$1; C=$2
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-graph"
$CMD > gpurun_out/ncu_plain_${TAG}.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo full rc=$?
