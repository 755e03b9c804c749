#!/bin/bash
# A/B of the x-run flux kernel (ADER_FLUX_RUNS=5..7: CTAs/SM of its register budget; 0 = default kernel)
mkdir -p gpurun_out
TAG=${1:-runs}
ADER_FLUX_RUNS=0 python tools/flux_ab.py save gpurun_out/fr_off.npz > gpurun_out/fr_off.log 2>&1 || tail gpurun_out/fr_off.log
ADER_FLUX_RUNS=7 python tools/flux_ab.py save gpurun_out/fr_on.npz > gpurun_out/fr_on.log 2>&1 || tail gpurun_out/fr_on.log
python tools/flux_ab.py cmp gpurun_out/fr_off.npz gpurun_out/fr_on.npz | tee gpurun_out/flux_runs_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/fr_*.npz
B="python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"; }
for v in 0 7 6 5 0 7; do
  ADER_FLUX_RUNS=$v timeout 600 $B > gpurun_out/b_${TAG}_$v.log 2>&1; show gpurun_out/b_${TAG}_$v.log "runs=$v c4"
done
