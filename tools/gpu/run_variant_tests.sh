#!/bin/bash
# a build variant through the capped / parity GPU tests, then its A/B lines:
# V=pdl CONFIGS="5 2" bash tools/gpu/run_variant_tests.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
MSURF_LIB=build_variants/$V.so timeout 900 python -m pytest tests/test_gpu_capped.py tests/test_gpu_configs.py -x -q > gpurun_out/vt_$V.log 2>&1; echo "rc=$?" >> gpurun_out/vt_$V.log
TAG=vt VARIANTS="$V" CONFIGS="${CONFIGS:-5 2}" bash tools/gpu/run_ab.sh
MSURF_LIB=build_variants/$V.so timeout 600 python tools/gpu/project_strips.py --configs 5 --ns 8 --steps 3 > gpurun_out/vt_${V}_proj.jsonl 2>/dev/null
