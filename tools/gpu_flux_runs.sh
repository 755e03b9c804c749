#!/bin/bash
# A/B of the x runs of k_face_flux_cells (ADER_FLUX_RL=1: off): bitwise F / u, then C4 / C2 bench
mkdir -p gpurun_out
TAG=${1:-runs}
ADER_FLUX_RL=1 python tools/flux_ab.py save gpurun_out/fr_off.npz > gpurun_out/fr_off.log 2>&1 || tail gpurun_out/fr_off.log
python tools/flux_ab.py save gpurun_out/fr_on.npz > gpurun_out/fr_on.log 2>&1 || tail gpurun_out/fr_on.log
python tools/flux_ab.py cmp gpurun_out/fr_off.npz gpurun_out/fr_on.npz | tee gpurun_out/flux_runs_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/fr_*.npz
B="python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"; }
for v in "1 0" "8 0" "8 6" "8 5" "1 0" "8 0"; do
  set -- $v
  ADER_FLUX_RL=$1 ADER_FLUX_MINB=$2 timeout 600 $B > gpurun_out/b_${TAG}_rl$1_mb$2.log 2>&1; show gpurun_out/b_${TAG}_rl$1_mb$2.log "rl=$1 minb=$2 c4"
done
for x in 1 8; do
ADER_FLUX_RL=$x timeout 600 python bench.py --config c2 --n 512 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c2_$x.log 2>&1; show gpurun_out/b_${TAG}_c2_$x.log "rl=$x c2"
done
ADER_FLUX_RL=1 timeout 600 python bench.py --config c4 --n 128 --flux osher --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_osh_1.log 2>&1; show gpurun_out/b_${TAG}_osh_1.log "rl=1 osher128"
timeout 600 python bench.py --config c4 --n 128 --flux osher --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_osh_8.log 2>&1; show gpurun_out/b_${TAG}_osh_8.log "rl=8 osher128"
