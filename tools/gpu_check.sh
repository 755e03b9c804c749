#!/bin/bash
# One gpurun session: smoke, GPU tests, short benches (outputs under gpurun_out/)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/gpu.txt 2>&1
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --n 256 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
tail -2 gpurun_out/bench_c2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -2 gpurun_out/bench_c4.log
