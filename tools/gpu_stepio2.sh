#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-io}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_step_io.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log; grep -E "^E  " gpurun_out/pytest_$TAG.log | head
for c in c4 c2; do
  if [ $c = c4 ]; then A=""; else A="--config c2 --n 512"; fi
  timeout 900 python bench.py $A --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.log 2>&1; tail -1 gpurun_out/bench_${TAG}_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
done
