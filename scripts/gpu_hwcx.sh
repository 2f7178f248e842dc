#!/bin/bash
# HWC exchange kernel: parity tests, then full-image HWC vs planar (and the tile kernel via L3_HWC_TILE=1).
TAG=${TAG:-hx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hwc or predictor_h2 or fault" > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for o in f32 u8; do
  for cfg in c3_cityscapes c2_imagenet; do
    crop=256x256; [ $cfg = c3_cityscapes ] && crop=512x1024
    timeout 300 python bench.py --config $cfg --crop $crop --layout chw --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('xchg', '$cfg', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'])" || tail -5 gpurun_out/${TAG}.err
    L3_HWC_TILE=1 timeout 300 python bench.py --config $cfg --crop $crop --layout chw --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('tile', '$cfg', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'])" || tail -5 gpurun_out/${TAG}.err
  done
done
