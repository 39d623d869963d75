set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python bench.py --steps 3 --warmup 2 --cpu-seconds 6 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
python bench.py --impl reference --steps 1 --warmup 0 --cpu-seconds 6 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?
tail -c 1500 gpurun_out/bench_ref.json
