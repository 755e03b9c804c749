#!/bin/bash
# GPU suite, then C4 bench A/B (default vs an env switch given as $2=VAR)
mkdir -p gpurun_out
TAG=${1:-x}; VAR=${2:-ADER_NO_FUSEZ}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
for mode in default switched default; do
  if [ $mode = switched ]; then export $VAR=1; else unset $VAR; fi
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$mode.log 2>&1; tail -1 gpurun_out/bench_${TAG}_$mode.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$mode', round(d['ms_per_step'],2), d['kernel_share_of_step'], round(d['roofline_kernels'][0]['frac'],3))"
done
