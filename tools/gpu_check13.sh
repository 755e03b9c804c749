#!/bin/bash
# full GPU suite, bench lines (C4 Rusanov, C4@128 Osher, C2@512), 256^3 launch list + ncu full captures
mkdir -p gpurun_out
TAG=${1:-r1final}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | grep -v "where\|+  " | head -10
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-400
timeout 900 python bench.py --n 128 --flux osher > gpurun_out/bench_c4_128_osher.log 2>&1; echo "bench c4 128 osher rc=$?"; tail -1 gpurun_out/bench_c4_128_osher.log | cut -c1-400
timeout 900 python bench.py --config c2 --n 512 > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"; tail -1 gpurun_out/bench_c2.log | cut -c1-400
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux|k_weno" -s 5 -c 5 -o gpurun_out/prof_${TAG}_c4_256 $CMD > gpurun_out/ncu_${TAG}_c4_256.log 2>&1; echo "ncu full rc=$?"
