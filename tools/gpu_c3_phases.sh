#!/bin/bash
# C3 (and C5) macro-step phases: bench line + ADER_AMR_TIMING host phase totals
mkdir -p gpurun_out
TAG=${1:-ph}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for c in c3 c5; do
ADER_AMR_TIMING=1 timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/ph_${TAG}_$c.log 2> gpurun_out/ph_${TAG}_$c.err; echo "$c rc=$?"
tail -1 gpurun_out/ph_${TAG}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernel_share_of_step'], d['gpu_launches'])"
grep -A12 "amr host" gpurun_out/ph_${TAG}_$c.err | head -30
done
nproc; lscpu | grep -E "Model name|MHz" | head -3
