#!/bin/bash
# Build a variant of libfs1.so with extra nvcc flags for A/B timing (select it with FS1_LIB).
# usage: bash tools/variant.sh NAME "-DFOO=1 -DBAR"   ->  gpurun_var/lib_NAME.so
N=$1; shift
mkdir -p gpurun_var/obj_$N
FS1_OBJ_DIR=gpurun_var/obj_$N FS1_BUILD_OUT=$PWD/gpurun_var/lib_$N.so FS1_NVCC_EXTRA="$*" \
  python -c "from paper_2202_10042_b200 import build; print(build.build())"
