#!/bin/bash
# ncu capture of the predictor and flux kernels on c4@128 and c2@512 (args: tag)
mkdir -p gpurun_out
TAG=${1:-x}
for CFG in "c4 128" "c2 512"; do
  set -- $CFG
  CMD="python bench.py --config $1 --n $2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
  timeout 600 $CMD > gpurun_out/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux" -s 2 -c 2 -o gpurun_out/prof_${TAG}_$1 $CMD > gpurun_out/ncu_${TAG}_$1.log 2>&1
  echo "ncu $1 rc=$?"
done
