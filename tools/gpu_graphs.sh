#!/bin/bash
# CUDA-graph uniform steps + rebalance by moved rows: tests, then C1/C2/C4 with and without graphs
mkdir -p gpurun_out
TAG=${1:-gr}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_step_io.py tests/test_gpu_multirank.py tests/test_gpu_host_comm.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_$TAG.log | head -10
for g in 0 1; do
  for c in c1 c2 c4; do
    case $c in c1) A="--config c1";; c2) A="--config c2 --n 512";; c4) A="";; esac
    ADER_NO_GRAPHS=$g timeout 900 python bench.py $A --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${TAG}_g${g}_$c.log 2>&1
    tail -1 gpurun_out/bench_${TAG}_g${g}_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('no_graphs=$g $c', round(d['ms_per_step'],4), '%.4g'%d['value'], 'launches', d['gpu_launches'], [(e['kernel'], round(e['frac'],3)) for e in d['roofline_kernels']])"
  done
done
