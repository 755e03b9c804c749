#!/bin/bash
# predictor contractions: warp shuffles (default build) vs shared memory (-DADER_PRED_SMEM), same box
mkdir -p gpurun_out
TAG=${1:-pab}
bench2() {
  for c in c4 c2; do
    if [ $c = c4 ]; then A=""; else A="--config c2 --n 512"; fi
    timeout 900 python bench.py $A --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_$1_$c.log 2>&1
    tail -1 gpurun_out/bench_${TAG}_$1_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 $c', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']], 'pw', round(d['pred_weno_fp64']['frac'],3))"
  done
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log; grep -E "^E  " gpurun_out/pytest_$TAG.log | head -5
timeout 600 python tools/pf_ab.py > gpurun_out/pf_ab_$TAG.log 2>&1; echo "pf_ab (walk uses smem contractions) rc=$?"; grep -c "bitwise=True" gpurun_out/pf_ab_$TAG.log
bench2 shfl
touch paper_1212_3585_b200/csrc/kernels.cu
make -s -C paper_1212_3585_b200/csrc NVCC="/usr/local/cuda/bin/nvcc -DADER_PRED_SMEM" > /dev/null 2>&1 || { echo smem build failed; exit 1; }
bench2 smem
