#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-900
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-1800
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -3 gpurun_out/bench_c5.log | cut -c1-1800
