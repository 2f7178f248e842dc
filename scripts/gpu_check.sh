#!/bin/bash
# Full GPU tests + bench lines for C3 fp32 / C3 u8 / C2 / C4 (one repetition).
TAG=${TAG:-chk}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
for leg in f32 u8 c2 c4; do
  case $leg in f32) a="";; u8) a="--out u8";; c2) a="--config c2_imagenet";; c4) a="--config c4_uhd";; esac
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 $a > gpurun_out/${TAG}_$leg.json 2>gpurun_out/${TAG}_$leg.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_$leg.json')); print('$leg', d['value'], d['ms_decode'], d['roofline']['frac'])" || tail -3 gpurun_out/${TAG}_$leg.err
done
