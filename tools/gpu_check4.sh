#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_amr.py -q -x > gpurun_out/pytest_amr.log 2>&1; echo "pytest amr rc=$?"
grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_amr.log | grep -v "where\|+  " | head -30
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_amr.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/pytest_gpu.log
