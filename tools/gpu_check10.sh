#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
bash tools/gpu_prof.sh ${1:-v6}
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-2500
timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"; tail -1 gpurun_out/bench_c2.log | cut -c1-700
