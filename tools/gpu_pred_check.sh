mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "one_step or 100_step" 2>&1 | tail -1
for r in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pr_c4_$r.log 2>&1
  grep '^{' gpurun_out/bench_pr_c4_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c4', d['ms_per_step'], '%.3g'%d['value'], d['kernel_share_of_step'])"
done
timeout 900 python bench.py --config c2 --n 512 --no-cpu-baseline > gpurun_out/bench_pr_c2.log 2>&1
grep '^{' gpurun_out/bench_pr_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c2', d['ms_per_step'], '%.3g'%d['value'])"
