set -x
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err; echo new rc=$?
grep -v "^frame" gpurun_out/c5_new.err | tail -12
MSURF_LIB=build_variants/libmsurf_head.so timeout 300 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c5_head.json 2> gpurun_out/c5_head.err; echo head rc=$?
grep -v "^frame" gpurun_out/c5_head.err | tail -5
