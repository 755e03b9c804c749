#!/bin/bash
# diagnose idle gaps in the timed region: a short GPU test run, then bench x3 with gap traces
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c4_256" > gpurun_out/gap_pytest.log 2>&1; echo "pytest rc=$?"
for i in 1 2 3; do
ADER_GAP_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/gap_$i.log 2>&1
grep -E "gap trace|step chunk" gpurun_out/gap_$i.log | tail -4
grep '^{' gpurun_out/gap_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('run $i', round(d['ms_per_step'],2), round(sum(d['kernel_share_of_step'].values()),3), d['e2e']['value'])"
done
uptime; ps aux --sort=-%cpu | head -8
