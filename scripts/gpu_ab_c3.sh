#!/bin/bash
# A/B of library variants on C3: fp32 (headline) and u8 narrow (crop bench full-decode leg), twice each.
TAG=${TAG:-abc3}
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  name=$(basename $lib .so)
  L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', 'c3 f32', d['value'], d['ms_decode'], d['roofline']['frac'])"
  L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --crop 512x1024 --out u8 --steps 100 > gpurun_out/${TAG}_tmp2.json 2>>gpurun_out/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp2.json')); print('$name', 'c3 u8 narrow full', d['ms_full_decode'])"
  if [ -n "${WITH_C4:-}" ]; then
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --config c4_uhd --no-cpu-baseline --e2e-steps 2 > gpurun_out/${TAG}_tmp3.json 2>>gpurun_out/${TAG}_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp3.json')); print('$name', 'c4 u8 wide', d['ms_decode'], d['roofline']['frac'])"
    L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --config c2_imagenet --no-cpu-baseline --e2e-steps 2 > gpurun_out/${TAG}_tmp4.json 2>>gpurun_out/${TAG}_${name}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp4.json')); print('$name', 'c2 u8', d['ms_decode'], d['roofline']['frac'])"
  fi
done
done
