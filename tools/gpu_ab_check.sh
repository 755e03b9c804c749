#!/bin/bash
# GPU suite, then C4 and C2 bench lines
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.log 2>&1; tail -1 gpurun_out/bench_${TAG}_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],2), d['kernel_share_of_step'], round(d['roofline_kernels'][0]['frac'],3), d['pred_sweeps_mean'])"
done
timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), d['kernel_share_of_step'], round(d['roofline']['frac'],3), d['pred_sweeps_mean'])"
