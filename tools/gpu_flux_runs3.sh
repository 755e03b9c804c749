B="python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"; }
for v in "8 5" "8 4" "16 5" "16 4" "8 5"; do
  set -- $v
  ADER_FLUX_RL=$1 ADER_FLUX_RUNS=$2 timeout 600 $B > gpurun_out/b_runs3_$1_$2.log 2>&1; show gpurun_out/b_runs3_$1_$2.log "rl=$1 mb=$2 c4"
done
