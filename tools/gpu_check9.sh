#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_amr.py -q -x > gpurun_out/pytest_amr.log 2>&1; echo "pytest amr rc=$?"; tail -2 gpurun_out/pytest_amr.log
grep -E "^FAILED|^E  " gpurun_out/pytest_amr.log | grep -v "where\|+  " | head -10
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"; tail -1 gpurun_out/bench_c3.log | cut -c1-1200
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-1200
