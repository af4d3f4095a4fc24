#!/bin/bash
# debug variant with per-phase clock64 counters (Eng::advance prints PHASES per instance)
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared -DSSB_PHASE_TIMING -I include -o tools/libssb_timing.so \
  paper_2410_17840_b200/csrc/ssb_kernels.cu paper_2410_17840_b200/csrc/ssb_summary.cu
