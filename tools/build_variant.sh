#!/bin/bash
# build an experimental libssb variant: tools/build_variant.sh NAME [extra nvcc flags...]
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared -I include "$@" -o tools/variants/libssb_$name.so \
  paper_2410_17840_b200/csrc/ssb_kernels.cu paper_2410_17840_b200/csrc/ssb_summary.cu 2>&1 | grep -v "spill\|^$"
