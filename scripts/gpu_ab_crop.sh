#!/bin/bash
# A/B of library variants on the crop bench (CHW layout; the old lib has no HWC flag).
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  name=$(basename $lib .so)
  for o in u8 f32; do
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --crop 512x1024 --out $o --steps 200 > gpurun_out/abc_tmp.json 2>gpurun_out/abc_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/abc_tmp.json')); print('$name', '$o', 'crop', d['ms_per_step'], 'full', d['ms_full_decode'])"
  done
done
done
