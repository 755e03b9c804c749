#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2e}
timeout 2400 python -m pytest tests/test_gpu_r2_configs.py tests/test_gpu_multirank.py -q -p no:randomly > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_$TAG.log
grep -E "^E  " gpurun_out/pytest_$TAG.log | head -20
