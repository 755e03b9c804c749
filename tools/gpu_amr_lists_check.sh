TAG=${1:-v20}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_amr.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -3
for c in c3 c6; do
ADER_AMR_TIMING=1 timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 --steps 5 > gpurun_out/amrt_${TAG:-v20}_$c.log 2>&1
grep -A3 "amr host" gpurun_out/amrt_${TAG:-v20}_$c.log | head -4
grep '^{' gpurun_out/amrt_${TAG:-v20}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c', d['ms_per_step'], d['value'], d['kernel_share_of_step'])"
done
