#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_amr.py::test_c3_full_size_first_macro_steps > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
timeout 600 python tools/explosion2d_probe.py > gpurun_out/probe2d.log 2>&1; echo "probe rc=$?"; cut -c1-250 gpurun_out/probe2d.log
bash tools/gpu_prof.sh ${1:-v5}
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-1500
