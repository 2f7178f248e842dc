#!/bin/bash
# HWC full-image A/B: the exchange kernel (default) vs the tile kernel (L3_HWC_TILE=1) per library, C3 and C2.
TAG=${TAG:-abh}
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  for o in f32 u8; do
    for cfg in c3_cityscapes c2_imagenet; do
      crop=256x256; [ $cfg = c3_cityscapes ] && crop=512x1024
      for tile in 0 1; do
        L3_HWC_TILE=$tile L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --config $cfg --crop $crop --layout chw --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
        python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', 'tile=$tile', '$cfg', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'])" || tail -5 gpurun_out/${TAG}.err
      done
    done
  done
done
