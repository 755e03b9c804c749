#!/bin/bash
# round 2: fused WENO + predictor (weno_pred.cu, ADER_WENO_PRED=1) — A/B (q, F, state)
# vs the separate kernels, uniform parity tests, C4 / C2 bench
mkdir -p gpurun_out
TAG=${1:-r2c}
timeout 600 python tools/flux_ab.py save /tmp/fa.npz && ADER_WENO_PRED=1 timeout 600 python tools/flux_ab.py save /tmp/fb.npz && python tools/flux_ab.py cmp /tmp/fa.npz /tmp/fb.npz > gpurun_out/fused_ab_$TAG.log 2>&1; echo "ab rc=$?"; tail -23 gpurun_out/fused_ab_$TAG.log
ADER_WENO_PRED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_$TAG.log
for L in 1 0; do
  ADER_WENO_PRED=$L timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_c4_fused$L.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_c4_fused$L.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('fused=$L c4', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'], [(k['kernel'], round(k.get('alu_tflops',0),2), round(k['frac'],3)) for k in d['roofline_kernels']])"
  ADER_WENO_PRED=$L timeout 600 python bench.py --config c2 --n 512 --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 1 > gpurun_out/bench_${TAG}_c2_fused$L.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_c2_fused$L.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('fused=$L c2', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'], [(k['kernel'], round(k.get('alu_tflops',0),2), round(k['frac'],3)) for k in d['roofline_kernels']])"
done
