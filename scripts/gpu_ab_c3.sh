#!/bin/bash
TAG=${TAG:-abc3}
for lib in "$@"; do
  name=$(basename $lib .so)
  L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', d['value'], d['ms_decode'], d['roofline']['frac'])"
done
