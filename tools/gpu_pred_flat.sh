#!/bin/bash
# A/B of the predictor's flat-cell first sweep (ADER_PRED_FLAT=0 switches it off): bitwise q / F / u, then C4 bench
mkdir -p gpurun_out
TAG=${1:-flat}
ADER_PRED_FLAT=0 python tools/flux_ab.py save gpurun_out/pf_off.npz > gpurun_out/pf_off.log 2>&1 || tail gpurun_out/pf_off.log
python tools/flux_ab.py save gpurun_out/pf_on.npz > gpurun_out/pf_on.log 2>&1 || tail gpurun_out/pf_on.log
python tools/flux_ab.py cmp gpurun_out/pf_off.npz gpurun_out/pf_on.npz | tee gpurun_out/pred_flat_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/pf_*.npz
B="python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],2), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],2)) for e in d['roofline_kernels']], d['pred_sweeps_mean'])"; }
for x in 0 1 0 1; do
ADER_PRED_FLAT=$x timeout 600 $B > gpurun_out/b_${TAG}_$x.log 2>&1; show gpurun_out/b_${TAG}_$x.log "flat=$x c4"
done
for x in 0 1; do
ADER_PRED_FLAT=$x timeout 600 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c3_$x.log 2>&1; show gpurun_out/b_${TAG}_c3_$x.log "flat=$x c3"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amr.py tests/test_gpu_pred_variants.py -q -x -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
