#!/bin/bash
# A/B of the flat cells without a q block (ADER_PRED_FLAT_SKIP=0: every block written and read)
mkdir -p gpurun_out
TAG=${1:-fs}
ADER_PRED_FLAT_SKIP=0 python tools/flux_ab.py save gpurun_out/fs_off.npz > gpurun_out/fs_off.log 2>&1 || tail gpurun_out/fs_off.log
python tools/flux_ab.py save gpurun_out/fs_on.npz > gpurun_out/fs_on.log 2>&1 || tail gpurun_out/fs_on.log
python tools/flux_ab.py cmp gpurun_out/fs_off.npz gpurun_out/fs_on.npz | tee gpurun_out/flat_skip_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/fs_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], [(e['kernel'], e['bound'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']], d.get('pred_flat_frac'))"; }
for x in 0 1 0 1; do
ADER_PRED_FLAT_SKIP=$x timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/b_${TAG}_$x.log 2>&1; show gpurun_out/b_${TAG}_$x.log "skip=$x c4"
done
for x in 0 1; do
ADER_PRED_FLAT_SKIP=$x timeout 600 python bench.py --n 128 --flux osher --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_osh_$x.log 2>&1; show gpurun_out/b_${TAG}_osh_$x.log "skip=$x osher128"
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_io.py tests/test_gpu_multirank.py tests/test_gpu_pred_variants.py tests/test_gpu_r2_configs.py -q -x -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
