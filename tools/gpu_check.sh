#!/bin/bash
# build, full GPU suite, C4 (x2) and C2 512^2 bench lines
mkdir -p gpurun_out
TAG=${1:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
fi
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_c4_$i.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c4_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],2), {k:v for k,v in d['kernel_share_of_step'].items() if v}, [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],2)) for e in d['roofline_kernels']], d['pred_sweeps_mean'])"
done
timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), {k:v for k,v in d['kernel_share_of_step'].items() if v}, [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']], round(d['pred_weno_fp64']['frac'],3), d['pred_sweeps_mean'])"
