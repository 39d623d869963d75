# batched (config 3) e2e breakdown + GPU tests + bench lines
set -x
CONFIGS="3 2" bash tools/gpu/run_iter.sh
timeout 300 python tools/gpu/e2e_profile3.py > gpurun_out/e2e3.log 2>&1; echo e2e rc=$?
head -20 gpurun_out/e2e3.log
