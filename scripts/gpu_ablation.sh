#!/bin/bash
# f2: ablation parity tests + the Fig. 10 bars on HD / FHD / C3 / UHD (one GPU).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ablation or encoder or original_paeth" 2>&1 | tail -5
for c in ${CONFIGS:-ab_hd ab_fhd c3_cityscapes c4_uhd}; do
  timeout 300 python bench.py --ablation --config $c --steps 5 > gpurun_out/ablation_$c.json 2> gpurun_out/ablation_$c.err || tail -5 gpurun_out/ablation_$c.err
  cat gpurun_out/ablation_$c.json
done
