#!/bin/bash
# GPU suite + C4 bench x2 + C3 with host-phase timers
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.log 2>&1; tail -1 gpurun_out/bench_${TAG}_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4 run $i', round(d['ms_per_step'],2), d['kernel_share_of_step'])"
done
ADER_AMR_TIMING=1 timeout 600 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/amrt_${TAG}_c3.log 2>&1; grep -A2 "amr host" gpurun_out/amrt_${TAG}_c3.log | head -3; grep '^{' gpurun_out/amrt_${TAG}_c3.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['ms_per_step'],3), d['value'])"
