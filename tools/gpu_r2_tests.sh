#!/bin/bash
# round 2: new GPU parity tests + AMR tests (margin, refine), then ncu of the fused kernel
mkdir -p gpurun_out
TAG=${1:-r2d}
timeout 2400 python -m pytest tests/test_gpu_r2_configs.py tests/test_gpu_amr.py -q -p no:randomly > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
if [ "${2:-}" = "ncu" ]; then
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ADER_WENO_PRED=1 $CMD > gpurun_out/plain_$TAG.log 2>&1 && ADER_WENO_PRED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_weno_predictor|k_predictor" -s 1 -c 1 -o gpurun_out/prof_${TAG}_fused $CMD > gpurun_out/ncu_${TAG}_fused.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predictor" -s 1 -c 1 -o gpurun_out/prof_${TAG}_pred $CMD > gpurun_out/ncu_${TAG}_pred.log 2>&1; echo "ncu2 rc=$?"
fi
