#!/bin/bash
# A/B of library variants: C3 fp32 decode time (and C3 u8 / C2 u8 for u_* variants), twice each.
TAG=${TAG:-abf}
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  name=$(basename $lib .so)
  case $name in
    u_*|base*) legs="f32 u8 c2" ;;
    *) legs="f32" ;;
  esac
  for leg in $legs; do
    case $leg in
      f32) args="" ;;
      u8) args="--out u8" ;;
      c2) args="--config c2_imagenet" ;;
    esac
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --steps 100 $args > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', '$leg', d['ms_decode'], d['roofline']['frac'])" || tail -3 gpurun_out/${TAG}_${name}.err
  done
done
done
