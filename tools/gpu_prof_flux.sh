#!/bin/bash
# ncu --set full of the face-flux kernel (new and legacy) at C4 256^3, one launch each
mkdir -p gpurun_out
TAG=${1:-r2a}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_face_flux -s 1 -c 1 -o gpurun_out/prof_${TAG}_flux $CMD > gpurun_out/ncu_${TAG}_flux.log 2>&1; echo "ncu rc=$?"
ADER_FLUX_LEGACY=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_face_flux -s 1 -c 1 -o gpurun_out/prof_${TAG}_fluxlegacy $CMD > gpurun_out/ncu_${TAG}_fluxlegacy.log 2>&1; echo "ncu legacy rc=$?"
