#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_amr.log 2>&1; echo "pytest amr rc=$?"; tail -2 gpurun_out/pytest_amr.log; grep -E "^FAILED|^E  " gpurun_out/pytest_amr.log | head -5
for cm in 200 0 1000 200 0; do
ADER_BENCH_CLOCK_MS=$cm timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/diag_$cm.log 2>&1; tail -1 gpurun_out/diag_$cm.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('clock_ms=$cm', round(d['ms_per_step'],2), round(sum(d['kernel_share_of_step'].values()),3))"
done
for c in c3 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/diag_$c.log 2>&1; tail -1 gpurun_out/diag_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), d['value'], d['kernel_share_of_step'])"; done
