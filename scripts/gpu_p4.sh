#!/bin/bash
# GPU check of the byte-form predictor: parity tests, then A/B of build_ab/*.so (two repetitions)
mkdir -p gpurun_out
TAG=${TAG:-p4}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -5 gpurun_out/${TAG}_pytest.log
TAG=${TAG}ab bash scripts/gpu_ab.sh "$@"
TAG=${TAG}ab bash scripts/gpu_ab.sh "$@"
