#!/bin/bash
# ncu --set full of one C2 512^2 predictor launch (step 5), env passed through (arg: tag)
mkdir -p gpurun_out
TAG=${1:-p}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_predictor" -s 5 -c 1 -o gpurun_out/prof_${TAG}_c2 python bench.py --config c2 --n 512 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${TAG}.log 2>&1; echo rc=$?
