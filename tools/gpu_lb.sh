#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-lb}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_host_comm.py tests/test_gpu_step_io.py -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_$TAG.log | cut -c1-200 | head -10
