#!/bin/bash
# bench lines of the remaining configs on the last build
mkdir -p gpurun_out
TAG=${1:-r2j}
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_${TAG}_$name.log 2>gpurun_out/bench_${TAG}_$name.err; echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_$name.log | cut -c1-130; }
run c2 --config c2 --n 512 ; run c3 --config c3 ; run c5 --config c5 ; run c4osher --n 128 --flux osher ; run c6 --config c6 --steps 5 --no-cpu-baseline ; run c1 --config c1 --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_reference.log 2>&1; echo "reference rc=$?"
