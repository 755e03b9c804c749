#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-awp}
ADER_AMR_WENO_PATCH=0 timeout 900 python tools/amr_weno_ab.py save gpurun_out/awp_off.npz 2>&1 | tail -6
timeout 900 python tools/amr_weno_ab.py save gpurun_out/awp_on.npz 2>&1 | tail -6
python tools/amr_weno_ab.py cmp gpurun_out/awp_off.npz gpurun_out/awp_on.npz | tee gpurun_out/amr_weno_cmp_$TAG.log
rm -f gpurun_out/awp_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), '%.4g'%d['value'], d['kernel_share_of_step'])"; }
for x in 0 1; do
ADER_AMR_WENO_PATCH=$x ADER_AMR_TIMING=1 timeout 900 python bench.py --config c6 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c6_$x.log 2>gpurun_out/b_${TAG}_c6_$x.err; show gpurun_out/b_${TAG}_c6_$x.log "patch=$x c6"
ADER_AMR_WENO_PATCH=$x timeout 900 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c3_$x.log 2>&1; show gpurun_out/b_${TAG}_c3_$x.log "patch=$x c3"
done
timeout 1800 python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py tests/test_gpu_r2_configs.py -q -x -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
