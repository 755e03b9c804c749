#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1 || exit 1
for r in 1 2; do for th in 1 64; do
  ADER_HOST_THREADS=$th timeout 900 python bench.py --config c3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3ab_${th}_$r.log 2>&1
  tail -1 gpurun_out/c3ab_${th}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads=$th', round(d['ms_per_step'],2))"
done; done
for th in 1 64; do ADER_HOST_THREADS=$th timeout 900 python bench.py --config c6 --steps 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c6ab_$th.log 2>&1; tail -1 gpurun_out/c6ab_$th.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c6 threads=$th', round(d['ms_per_step'],1))"; done
