#!/bin/bash
# AMR host path changes: AMR + multirank + host-comm suites, then C3 / C6 timing with phase breakdown
mkdir -p gpurun_out
TAG=${1:-ah}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py tests/test_gpu_host_comm.py tests/test_gpu_r2_configs.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_$TAG.log | head -10
bash tools/gpu_amr_phase_diff.sh c3
for i in 1 2; do timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3_$i.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c3_$i.log | cut -c1-250; done
timeout 900 python bench.py --config c6 --steps 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c6.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c6.log | cut -c1-250
