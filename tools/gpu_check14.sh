#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_multirank.log 2>&1; echo "pytest multirank rc=$?"; tail -3 gpurun_out/pytest_multirank.log
grep -E "^FAILED|^E  " gpurun_out/pytest_multirank.log | head -10
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_rep$i.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4_rep$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_share_of_step'])"
done
nvidia-smi --query-gpu=name,memory.used,memory.total,clocks.sm,clocks.max.sm,power.draw --format=csv
