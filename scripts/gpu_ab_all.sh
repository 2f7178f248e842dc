#!/bin/bash
# A/B of library variants on every planar config: C3 fp32, C3 u8, C2, C4, twice each (decode ms, roofline frac).
TAG=${TAG:-aba}
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  name=$(basename $lib .so)
  for leg in f32 u8 c2 c4; do
    case $leg in f32) a="";; u8) a="--out u8";; c2) a="--config c2_imagenet";; c4) a="--config c4_uhd";; esac
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --steps 100 $a > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', '$leg', d['ms_decode'], d['roofline']['frac'])" || tail -3 gpurun_out/${TAG}_${name}.err
  done
done
done
