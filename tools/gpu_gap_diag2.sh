#!/bin/bash
# catch an idle-gap run: bench x6 with gap traces (3 back to back, 3 after 30 s pauses)
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
  if [ $i -gt 3 ]; then sleep 30; fi
  ADER_GAP_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/gap2_$i.log 2>&1
  grep '^{' gpurun_out/gap2_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('run $i', round(d['ms_per_step'],2), round(sum(d['kernel_share_of_step'].values()),3), d['clocks'])"
  grep -E "gap trace|step chunk: 10" gpurun_out/gap2_$i.log | cut -c1-400
  nvidia-smi --query-compute-apps=pid,used_memory --format=csv,noheader | head -3
done
