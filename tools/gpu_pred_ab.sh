#!/bin/bash
# A/B of a predictor variant selected by an env var (arg 2, e.g. ADER_PRED_DMMA): q/state/cells and
# sweeps vs the variant switched off, then C2 and C5 bench lines both ways
mkdir -p gpurun_out
TAG=${1:-ab}; VAR=${2:-ADER_PRED_DMMA}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
env $VAR=0 timeout 600 python tools/pred_ab.py save gpurun_out/ab_off_$TAG.npz 2>&1 | tail -3
timeout 600 python tools/pred_ab.py save gpurun_out/ab_on_$TAG.npz 2>&1 | tail -3
python tools/pred_ab.py cmp gpurun_out/ab_off_$TAG.npz gpurun_out/ab_on_$TAG.npz
for x in 0 1 0 1; do
for c in "c2 --n 512" "c5"; do
env $VAR=$x timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_$x.log 2>&1; tail -1 gpurun_out/bench_${TAG}_$x.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$x', '$c', round(d['ms_per_step'],4), [(k['kernel'], round(k.get('ms_per_launch',0),4), round(k['frac'],3)) for k in d['roofline_kernels']], round(d['pred_weno_fp64']['frac'],3), d['pred_sweeps_mean'])"
done
done
