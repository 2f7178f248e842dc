#!/bin/bash
# Full GPU test suite (parity + sanitizers) on one B200.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build_smoke.log 2>&1 || { tail -20 gpurun_out/build_smoke.log; exit 1; }
tail -2 gpurun_out/build_smoke.log
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
