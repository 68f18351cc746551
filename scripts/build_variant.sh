#!/bin/bash
# Build a variant of the product library with extra nvcc flags for A/B timing:
#   scripts/build_variant.sh NAME -DFLAG ...  ->  scratch/libpipespec_NAME.so
# (select it with PS_LIB=scratch/libpipespec_NAME.so; scratch/ is git-ignored)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p scratch
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -cudart static "$@" -o scratch/libpipespec_$name.so paper_2505_01572_b200/csrc/ps_stage.cu paper_2505_01572_b200/csrc/ps_pipeline.cu
echo scratch/libpipespec_$name.so
