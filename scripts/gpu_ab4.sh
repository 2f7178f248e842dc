#!/bin/bash
# A/B of library variants (paths relative to the repo; "tree" = the in-tree build) on C3 f32, C3 u8,
# C2 u8 and C4 u8, REPS repetitions; then (if PARITY=1) the GPU parity suite on every variant.
mkdir -p gpurun_out
TAG=${TAG:-ab4}
CFGS=${CFGS:-"c3f32 c3u8 c2 c4"}
for rep in $(seq ${REPS:-2}); do
for lib in "$@"; do
  if [ "$lib" = tree ]; then L=$PWD/paper_2208_08711_b200/libl3_b200.so; name=tree; else L=$PWD/$lib; name=$(basename $lib .so); fi
  for c in $CFGS; do
    case $c in
      c3f32) a="--config c3_cityscapes" ;; c3u8) a="--config c3_cityscapes --out u8" ;;
      c2) a="--config c2_imagenet" ;; c4) a="--config c4_uhd" ;;
    esac
    L3_B200_LIB_OVERRIDE=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --steps ${STEPS:-100} $a > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}_$c.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', '$c', d['ms_decode'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
done
if [ -n "$PARITY" ]; then
  for lib in "$@"; do
    if [ "$lib" = tree ]; then L=$PWD/paper_2208_08711_b200/libl3_b200.so; else L=$PWD/$lib; fi
    L3_B200_LIB_OVERRIDE=$L timeout 1200 python -m pytest tests -m gpu -x -q ${PK:+-k "$PK"} 2>&1 | tail -3
  done
fi
