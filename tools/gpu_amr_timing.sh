#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-at}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
ADER_AMR_TIMING=1 timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.log 2>gpurun_out/bench_${TAG}_c3.err; echo "c3 rc=$?"
tail -1 gpurun_out/bench_${TAG}_c3.log | cut -c1-300; grep -A2 "amr host phases" gpurun_out/bench_${TAG}_c3.err | head -8
ADER_AMR_TIMING=1 timeout 900 python bench.py --config c6 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_c6.log 2>gpurun_out/bench_${TAG}_c6.err; echo "c6 rc=$?"
tail -1 gpurun_out/bench_${TAG}_c6.log | cut -c1-300; grep -A2 "amr host phases" gpurun_out/bench_${TAG}_c6.err | head -8
