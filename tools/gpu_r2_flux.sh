#!/bin/bash
# round 2: new face-flux kernel (flux_tma.cu) — bitwise A/B vs the round-1 kernel,
# uniform parity tests, C4 bench with both kernels
mkdir -p gpurun_out
TAG=${1:-r2a}
ADER_FLUX_LEGACY=1 timeout 600 python tools/flux_ab.py save /tmp/fa.npz && timeout 600 python tools/flux_ab.py save /tmp/fb.npz && python tools/flux_ab.py cmp /tmp/fa.npz /tmp/fb.npz > gpurun_out/flux_ab_$TAG.log 2>&1; echo "ab rc=$?"; cat gpurun_out/flux_ab_$TAG.log | tail -16
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_$TAG.log
for L in 0 1; do
  ADER_FLUX_LEGACY=$L timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_c4_legacy$L.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_c4_legacy$L.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('legacy=$L c4', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'], d['roofline'])"
done
