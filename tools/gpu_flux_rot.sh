#!/bin/bash
# A/B of the face-flux kernels: k_face_flux_cells (default) vs k_face_flux_rot (ADER_FLUX_ROT=1)
mkdir -p gpurun_out
TAG=${1:-rot}
python tools/flux_ab.py save gpurun_out/fab_base.npz > gpurun_out/fab_base.log 2>&1 || { echo base save failed; tail gpurun_out/fab_base.log; }
ADER_FLUX_ROT=1 python tools/flux_ab.py save gpurun_out/fab_rot.npz > gpurun_out/fab_rot.log 2>&1 || { echo rot save failed; tail gpurun_out/fab_rot.log; }
ADER_FLUX_ROT=1 ADER_FLUX_RL=4 ADER_FLUX_MINB=3 python tools/flux_ab.py save gpurun_out/fab_rot1.npz > gpurun_out/fab_rot1.log 2>&1
python tools/flux_ab.py cmp gpurun_out/fab_base.npz gpurun_out/fab_rot.npz | tee gpurun_out/fab_cmp_$TAG.log
python tools/flux_ab.py cmp gpurun_out/fab_rot.npz gpurun_out/fab_rot1.npz | tee gpurun_out/fab_cmp1_$TAG.log
rm -f gpurun_out/fab_*.npz
B="python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],2), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],2)) for e in d['roofline_kernels']])"; }
timeout 600 $B > gpurun_out/b_${TAG}_base.log 2>&1; show gpurun_out/b_${TAG}_base.log base
for v in "8 16 5" "8 16 4" "8 16 3" "4 16 4" "8 4 4" "8 8 3"; do
  set -- $v
  ADER_FLUX_ROT=1 ADER_FLUX_RL=$1 ADER_FLUX_YC=$2 ADER_FLUX_MINB=$3 timeout 600 $B > gpurun_out/b_${TAG}_rl$1_yc$2_mb$3.log 2>&1
  show gpurun_out/b_${TAG}_rl$1_yc$2_mb$3.log "rot rl=$1 yc=$2 minb=$3"
done
ADER_FLUX_ROT=1 timeout 600 python bench.py --config c2 --n 512 --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_c2rot.log 2>&1; show gpurun_out/b_${TAG}_c2rot.log c2rot
timeout 600 python bench.py --config c2 --n 512 --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b_${TAG}_c2base.log 2>&1; show gpurun_out/b_${TAG}_c2base.log c2base
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ADER_FLUX_ROT=1 ADER_NO_GRAPHS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_face_flux" -s 4 -c 1 -o gpurun_out/prof_${TAG}_flux $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
