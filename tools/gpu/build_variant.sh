# build_variant.sh NAME "-DFLAGS..." -> build_variants/libmsurf_NAME.so (same flags as build())
NAME=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -shared \
  -Xcompiler -fPIC,-ffp-contract=off,-fno-fast-math -I include "$@" -o build_variants/libmsurf_$NAME.so \
  paper_2603_28160_b200/csrc/msurf.cu paper_2603_28160_b200/csrc/msurf_plan.cpp 2>&1 | grep -A2 "sweep_kernelILi[0-9]ELb0" | grep "Used\|spill" | head -12
