# AMR tests + smoke + the AMR bench lines (e2e includes ader_get_cells every step)
TAG=${1:-gc}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for c in c5 c3 c6; do
  ex=""; [ $c = c6 ] && ex="--steps 5 --no-cpu-baseline"
  timeout 900 python bench.py --config $c $ex > gpurun_out/bench_${TAG}_$c.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c', d['ms_per_step'], '%.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'])"
done
