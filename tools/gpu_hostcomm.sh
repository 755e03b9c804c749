#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-hc}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_host_comm.py -q -x -s > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  |Error" gpurun_out/pytest_$TAG.log | head -20
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest2_$TAG.log 2>&1; echo "pytest2 rc=$?"; tail -2 gpurun_out/pytest2_$TAG.log
