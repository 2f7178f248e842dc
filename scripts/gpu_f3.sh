#!/bin/bash
# f3: crop / flip / HWC parity + the partial-decode and HWC timings on C3 (one GPU).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "crop or hwc or fault" 2>&1 | tail -3
for o in u8 f32; do for l in chw hwc; do
  timeout 300 python bench.py --crop 512x1024 --layout $l --out $o --steps 50 > gpurun_out/crop_${o}_${l}.json 2> gpurun_out/crop_${o}_${l}.err || tail -5 gpurun_out/crop_${o}_${l}.err
  cat gpurun_out/crop_${o}_${l}.json
done; done
