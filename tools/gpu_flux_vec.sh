#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-fv}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_io.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
grep -E "^E  " gpurun_out/pytest_$TAG.log | head
timeout 600 python tools/pf_ab.py > gpurun_out/pf_ab_$TAG.log 2>&1; echo "pf_ab rc=$?"; tail -2 gpurun_out/pf_ab_$TAG.log
for i in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_c4_$i.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c4_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],2), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],2)) for e in d['roofline_kernels']], 'e2e %.4g'%d['e2e']['value'])"
done
timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.log 2>&1; tail -1 gpurun_out/bench_${TAG}_c2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_face_flux" -s 4 -c 1 -o gpurun_out/prof_${TAG}_flux $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
