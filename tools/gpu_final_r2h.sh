#!/bin/bash
# final evidence after the x-run flux kernel: full GPU suite, smoke, C4 bench lines (default K and the 50 steps of
# BASELINE configs[3]), launch list and ncu --set full of a timed C4 step
mkdir -p gpurun_out
TAG=${1:-r2h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_${TAG}_$name.log 2>gpurun_out/bench_${TAG}_$name.err; echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_$name.log | cut -c1-160; }
run c4 ; run c4b ; run c4_50steps --steps 50 --warmup 3 --no-cpu-baseline
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux|k_weno|k_update" -s 24 -c 6 -o gpurun_out/prof_${TAG}_c4_step5 $CMD > gpurun_out/ncu_${TAG}_c4.log 2>&1; echo "ncu c4 rc=$?"
