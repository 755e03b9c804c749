#!/bin/bash
# fused walk: A/B bitwise check + ncu --set full of one walk launch at C4 256^3
mkdir -p gpurun_out
TAG=${1:-pfp}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python tools/pf_ab.py > gpurun_out/pf_ab_$TAG.log 2>&1; echo "pf_ab rc=$?"; tail -40 gpurun_out/pf_ab_$TAG.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pred_flux" -s 4 -c 1 -o gpurun_out/prof_${TAG}_walk $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
