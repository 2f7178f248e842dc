#!/bin/bash
# A/B of library variants on C4 (u8, wide 8-column path), twice each.
TAG=${TAG:-ab4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or c4 or fault" > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
for lib in "$@"; do
  name=$(basename $lib .so)
  L3_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --config c4_uhd --no-cpu-baseline --e2e-steps 2 --steps 100 > gpurun_out/${TAG}_tmp.json 2>gpurun_out/${TAG}_${name}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_tmp.json')); print('$name', 'c4', d['ms_decode'], d['roofline']['frac'])" || tail -3 gpurun_out/${TAG}_${name}.err
done
done
