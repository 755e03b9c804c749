#!/bin/bash
# A/B of the AMR face flux with the face lookups spread over lanes against the previous build
# (paper_1212_3585_b200/libader_b200_prev.so): cells bitwise, C6 / C3 / C5 bench
mkdir -p gpurun_out
TAG=${1:-afl}
ADER_AB_LIB=$PWD/paper_1212_3585_b200/libader_b200_prev.so timeout 900 python tools/amr_weno_ab.py save gpurun_out/afl_prev.npz 2>&1 | tail -2
timeout 900 python tools/amr_weno_ab.py save gpurun_out/afl_new.npz 2>&1 | tail -2
python tools/amr_weno_ab.py cmp gpurun_out/afl_prev.npz gpurun_out/afl_new.npz | tee gpurun_out/amr_flux_cmp_$TAG.log
rm -f gpurun_out/afl_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), '%.4g'%d['value'], d['kernel_share_of_step'])"; }
ADER_AMR_TIMING=1 timeout 900 python bench.py --config c6 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c6.log 2>gpurun_out/b_${TAG}_c6.err; show gpurun_out/b_${TAG}_c6.log "c6"
timeout 900 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c3.log 2>&1; show gpurun_out/b_${TAG}_c3.log "c3"
timeout 900 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c3b.log 2>&1; show gpurun_out/b_${TAG}_c3b.log "c3"
timeout 900 python bench.py --config c5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c5.log 2>&1; show gpurun_out/b_${TAG}_c5.log "c5"
timeout 1800 python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py -q -x -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
