#!/bin/bash
# full GPU suite, C4 bench with the line-walker flux kernel and the cell-per-warp one, ncu of both
mkdir -p gpurun_out
TAG=${1:-v12}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
for K in cells lines; do
ADER_FLUX_KERNEL=$K timeout 900 python bench.py > gpurun_out/bench_c4_${TAG}_$K.log 2>&1; echo "bench c4 $K rc=$?"; tail -1 gpurun_out/bench_c4_${TAG}_$K.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['kernel_share_of_step'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['achieved'])"
done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ADER_FLUX_KERNEL=lines timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_face_flux" -s 1 -c 1 -o gpurun_out/prof_${TAG}_lines $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
