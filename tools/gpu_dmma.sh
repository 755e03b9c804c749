#!/bin/bash
# DMMA throughput microbenchmark + ncu of the C2 predictor (is it shared-memory bound?)
mkdir -p gpurun_out
TAG=${1:-dm}
true
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config c2 --n 512 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predictor" -s 3 -c 1 -o gpurun_out/prof_${TAG}_c2pred $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
