#!/bin/bash
# fused predictor + face-flux walk: bitwise A/B vs the separate kernels, then C4 / C2 timing both ways
mkdir -p gpurun_out
TAG=${1:-pf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python tools/pf_ab.py > gpurun_out/pf_ab_$TAG.log 2>&1; echo "pf_ab rc=$?"; tail -40 gpurun_out/pf_ab_$TAG.log
for fuse in 0 1; do
  ADER_FUSE_PRED_FLUX=$fuse timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_c4_fuse$fuse.log 2>&1; echo "c4 fuse=$fuse rc=$?"
  tail -1 gpurun_out/bench_${TAG}_c4_fuse$fuse.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],2), d['kernel_share_of_step'], d['pred_sweeps_mean'])"
  ADER_FUSE_PRED_FLUX=$fuse timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_c2_fuse$fuse.log 2>&1; echo "c2 fuse=$fuse rc=$?"
  tail -1 gpurun_out/bench_${TAG}_c2_fuse$fuse.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), d['kernel_share_of_step'], d['pred_sweeps_mean'])"
done
