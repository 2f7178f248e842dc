#!/bin/bash
# End-of-round-2 refresh: the full GPU tests + smoke, then the measurement session (scripts/gpu_round2.sh).
mkdir -p gpurun_out
TAG=${TAG:-r2b}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
TAG=$TAG bash scripts/gpu_round2.sh
