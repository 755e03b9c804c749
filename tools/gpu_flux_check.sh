# flux-kernel change: uniform parity + multirank tests, C4 / Osher bench lines
TAG=${1:-fx}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
for r in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_c4_$r.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_c4_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c4', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'])"
done
timeout 900 python bench.py --n 128 --flux osher --no-cpu-baseline > gpurun_out/bench_${TAG}_osher.log 2>&1
grep '^{' gpurun_out/bench_${TAG}_osher.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('osher', d['ms_per_step'], '%.3g'%d['value'])"
