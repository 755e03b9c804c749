#!/bin/bash
# round 2: face-flux walk kernel (flux_tma.cu, ADER_FLUX_TMA=1) — A/B vs the round-1
# kernel, uniform parity tests, C4 bench with both kernels (+ optional ncu of the new one)
mkdir -p gpurun_out
TAG=${1:-r2b}
timeout 600 python tools/flux_ab.py save /tmp/fa.npz && ADER_FLUX_TMA=1 timeout 600 python tools/flux_ab.py save /tmp/fb.npz && python tools/flux_ab.py cmp /tmp/fa.npz /tmp/fb.npz > gpurun_out/flux_ab_$TAG.log 2>&1; echo "ab rc=$?"; tail -16 gpurun_out/flux_ab_$TAG.log
ADER_FLUX_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_$TAG.log
for L in 1 0; do
  ADER_FLUX_TMA=$L timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_c4_tma$L.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_c4_tma$L.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('tma=$L c4', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'], d['roofline']['achieved'], d['roofline']['frac'])"
done
if [ "${2:-}" = "ncu" ]; then
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
ADER_FLUX_TMA=1 $CMD > gpurun_out/plain_$TAG.log 2>&1 && ADER_FLUX_TMA=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_face_flux -s 1 -c 1 -o gpurun_out/prof_${TAG}_flux $CMD > gpurun_out/ncu_${TAG}_flux.log 2>&1; echo "ncu rc=$?"
fi
