#!/bin/bash
# full GPU suite, two C4 bench lines, ncu --set full of the WENO sweeps and the face flux at 256^3 (arg: tag)
mkdir -p gpurun_out
TAG=${1:-v10}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
for i in 1 2; do
timeout 900 python bench.py > gpurun_out/bench_c4_$TAG_$i.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4_$TAG_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['kernel_share_of_step'], d['roofline']['kernel'], d['roofline']['frac'])"
done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_weno|k_predictor|k_face_flux" -s 5 -c 5 -o gpurun_out/prof_${TAG}_c4_256 $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
