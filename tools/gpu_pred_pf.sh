#!/bin/bash
# A/B of the predictor's L2 prefetch distance (ADER_PRED_PF)
mkdir -p gpurun_out
TAG=${1:-pf}
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']], d['pred_sweeps_mean'])"; }
for x in 0 2 1 4 8 0 2; do
ADER_PRED_PF=$x timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_$x.log 2>&1; show gpurun_out/b_${TAG}_$x.log "pf=$x c4"
done
for x in 0 2 4; do
ADER_PRED_PF=$x timeout 600 python bench.py --config c2 --n 512 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c2_$x.log 2>&1; show gpurun_out/b_${TAG}_c2_$x.log "pf=$x c2"
done
