#!/bin/bash
# HWC exchange kernel A/B: full-image HWC time (crop bench's ms_full_decode_hwc) per library variant.
TAG=${TAG:-abx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hwc or predictor_h2 or fault" > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
for lib in "$@"; do
  name=$(basename $lib .so)
  for o in f32 u8; do
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --crop 512x1024 --layout chw --out $o --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', '$o', 'planar', d['ms_full_decode'], 'hwc', d['ms_full_decode_hwc'])" || tail -5 gpurun_out/${TAG}.err
  done
done
