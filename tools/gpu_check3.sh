#!/bin/bash
# bench + ncu evidence for the default workload (outputs under gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "c4_256 or explosion" > gpurun_out/pytest_c4.log 2>&1; echo "pytest c4 rc=$?"; tail -3 gpurun_out/pytest_c4.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-3000
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_predictor -s 2 -c 1 -o gpurun_out/prof_pred $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_face_flux -s 1 -c 1 -o gpurun_out/prof_flux $CMD > gpurun_out/ncu_full_flux.log 2>&1
echo "ncu flux rc=$?"
