#!/bin/bash
# A/B of the WENO sweeps' 3D-grid indexing (ADER_WENO_G3=0: linear index decomposed by division)
mkdir -p gpurun_out
TAG=${1:-g3}
ADER_WENO_G3=0 python tools/flux_ab.py save gpurun_out/g3_off.npz > gpurun_out/g3_off.log 2>&1 || tail gpurun_out/g3_off.log
python tools/flux_ab.py save gpurun_out/g3_on.npz > gpurun_out/g3_on.log 2>&1 || tail gpurun_out/g3_on.log
python tools/flux_ab.py cmp gpurun_out/g3_off.npz gpurun_out/g3_on.npz | tee gpurun_out/weno_g3_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/g3_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), d['kernel_share_of_step']['weno_reconstruct'], round(d['kernel_share_of_step']['weno_reconstruct']*d['ms_per_step'],3), 'ms weno')"; }
for x in 0 1 0 1; do
ADER_WENO_G3=$x timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_c4_$x.log 2>&1; show gpurun_out/b_${TAG}_c4_$x.log "g3=$x c4"
ADER_WENO_G3=$x timeout 600 python bench.py --config c2 --n 512 --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_c2_$x.log 2>&1; show gpurun_out/b_${TAG}_c2_$x.log "g3=$x c2"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_io.py tests/test_gpu_multirank.py -q -x -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
