#!/bin/bash
# Build an A/B variant of the decode library into build_ab/NAME.so with extra -D flags, e.g.
#   bash scripts/build_variant.sh es1 -DL3_EDGE_SEL=1
#   TAG=x bash scripts/gpu_ab.sh paper_2208_08711_b200/libl3_b200.so build_ab/es1.so   (under gpurun)
# Flags (l3_decode_fast.cuh / l3_decode_wide8.cuh): L3_PRED4, L3_PRED4_WIDE, L3_EDGE_SEL,
# L3_SMEM_PREFIX, L3_MIN_CTAS. `python scripts/sass_loops.py build_ab/NAME.so` shows the row loops.
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build_ab
timeout 900 /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared --expt-relaxed-constexpr -I include "$@" -o build_ab/$name.so paper_2208_08711_b200/csrc/*.cu
echo build_ab/$name.so
