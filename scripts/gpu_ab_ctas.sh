#!/bin/bash
for c in 6 5 4 3; do
  for cfg in "--config c3_cityscapes" "--config c3_cityscapes --out u8" "--config c4_uhd" "--config c2_imagenet"; do
    L3_DEV_CTAS_PER_SM=$c timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 $cfg > gpurun_out/abc_tmp.json 2>gpurun_out/abc.err
    python -c "import json; d=json.load(open('gpurun_out/abc_tmp.json')); print('ctas=$c', '$cfg', d['value'], d['ms_decode'], d['roofline']['frac'])"
  done
done
