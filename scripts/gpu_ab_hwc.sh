#!/bin/bash
# A/B of HWC kernel variants (libs as args): full-image HWC decode of C3, u8 and f32.
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  for o in f32 u8; do
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --crop 1024x2048 --layout hwc --out $o --steps 100 > gpurun_out/abh_tmp.json 2>gpurun_out/abh_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/abh_tmp.json')); print('$name', '$o', 'full_hwc', d['ms_full_decode_hwc'], 'chw', d['ms_full_decode'])"
  done
done
