#!/bin/bash
# f32 narrow vs f32 wide (L3_B200_FORCE_WIDE) on C3 / C4
for cfg in "--config c3_cityscapes" "--config c4_uhd --out f32" ; do
  for w in 0 1; do
    L3_FORCE_WIDE=$w timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 $cfg > gpurun_out/abw_tmp.json 2>gpurun_out/abw.err
    python -c "import json; d=json.load(open('gpurun_out/abw_tmp.json')); print('wide=$w', '$cfg', d['value'], d['ms_decode'], d['roofline']['frac'])"
  done
done
