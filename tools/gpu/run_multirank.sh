# functional check of the N>1 bench paths with 2 ranks on one GPU (gloo)
set -x
MSURF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_c2.json 2> gpurun_out/mr_c2.err; echo c2 rc=$?
tail -c 1500 gpurun_out/mr_c2.json; tail -5 gpurun_out/mr_c2.err
MSURF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config 3 --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_c3.json 2> gpurun_out/mr_c3.err; echo c3 rc=$?
tail -c 600 gpurun_out/mr_c3.json; tail -5 gpurun_out/mr_c3.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --cpu-seconds 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
tail -c 300 gpurun_out/mr_ref.json
