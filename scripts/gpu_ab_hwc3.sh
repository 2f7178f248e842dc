#!/bin/bash
# HWC A/B per library: full-image HWC and 512x1024 crop HWC (C3 fp32 / u8), full HWC on C2; parity of the first lib.
TAG=${TAG:-abh3}
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hwc or crop" > gpurun_out/${TAG}_${name}_pytest.log 2>&1; echo $name $(tail -1 gpurun_out/${TAG}_${name}_pytest.log)
  for o in f32 u8; do
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --crop 512x1024 --layout hwc --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', 'c3', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'], 'crop_hwc', d['ms_per_step'])" || tail -5 gpurun_out/${TAG}.err
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --config c2_imagenet --crop 256x256 --layout hwc --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', 'c2', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'], 'crop_hwc', d['ms_per_step'])" || tail -5 gpurun_out/${TAG}.err
  done
done
