#!/bin/bash
# round-end evidence: full GPU suite, bench lines of every BASELINE config + Osher,
# ncu launch list of the default bench command, ncu --set full of the hot kernels at 256^3
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu_$TAG.log | grep -v "where\|+  " | head -10
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_${TAG}_$name.log 2>&1; echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_$name.log | cut -c1-300; }
run c4 ; run c4b ; run c2 --config c2 --n 512 ; run c3 --config c3 ; run c5 --config c5 ; run c4osher --n 128 --flux osher ; run c6 --config c6 --steps 5 --no-cpu-baseline
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_reference.log 2>&1; echo "reference rc=$?"; tail -1 gpurun_out/bench_${TAG}_reference.log | cut -c1-300
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux|k_weno|k_update" -s 6 -c 6 -o gpurun_out/prof_${TAG}_c4_256 $CMD > gpurun_out/ncu_${TAG}_c4_256.log 2>&1; echo "ncu full rc=$?"
