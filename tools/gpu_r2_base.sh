#!/bin/bash
# round-2 baseline evidence: full GPU suite, smoke, default bench, clocked FP64 peak, launch list
mkdir -p gpurun_out
TAG=${1:-r2base}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c4.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}_c4.log | cut -c1-400
bash tools/gpu_fp64_peak.sh
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
