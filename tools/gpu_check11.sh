#!/bin/bash
# GPU check: full -m gpu suite, C4 bench with both fluxes, ncu capture of the Osher flux kernel
mkdir -p gpurun_out
TAG=${1:-v9}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-2500
timeout 900 python bench.py --flux osher > gpurun_out/bench_c4_osher.log 2>&1; echo "bench c4 osher rc=$?"; tail -1 gpurun_out/bench_c4_osher.log | cut -c1-2500
CMD="python bench.py --config c4 --n 128 --flux osher --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_osher.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_face_flux" -s 1 -c 1 -o gpurun_out/prof_${TAG}_osher $CMD > gpurun_out/ncu_${TAG}_osher.log 2>&1
echo "ncu osher rc=$?"
