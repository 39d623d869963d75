#!/bin/bash
# functional check of the N>1 bench paths with 2 ranks on one GPU (gloo: NCCL needs one GPU per rank)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
MSURF_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_c5.json 2> gpurun_out/mr_c5.err; echo c5 rc=$?
MSURF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config 2 --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_c2.json 2> gpurun_out/mr_c2.err; echo c2 rc=$?
MSURF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --config 3 --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mr_c3.json 2> gpurun_out/mr_c3.err; echo c3 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --cpu-seconds 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
# --gpus 2 without torchrun on a 1-GPU box must refuse loudly
timeout 120 python bench.py --gpus 2 --steps 1 --warmup 0 > gpurun_out/mr_spawn.json 2> gpurun_out/mr_spawn.err; echo spawn rc=$?
timeout 1200 python tools/gpu/project_strips.py --configs 5 2 4 > gpurun_out/project_r2b.jsonl 2> gpurun_out/project_r2b.err; echo proj rc=$?
