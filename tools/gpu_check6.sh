#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
bash tools/gpu_prof.sh ${1:-v3}
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-1500
