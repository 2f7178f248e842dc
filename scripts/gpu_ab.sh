#!/bin/bash
# A/B of library variants: L3 libs given as args (paths relative to repo)
mkdir -p gpurun_out
TAG=${TAG:-ab}
for lib in "$@"; do
  name=$(basename $lib .so)
  for cfg in "--config c3_cityscapes" "--config c3_cityscapes --out u8" "--config c2_imagenet" "--config c4_uhd"; do
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 $cfg > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', '$cfg', d['value'], d['ms_decode'], d['roofline']['frac'])"
  done
done
