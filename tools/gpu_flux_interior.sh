#!/bin/bash
# A/B of the interior fast path of the x-run flux kernel against the previous build (libader_b200_prev.so)
mkdir -p gpurun_out
TAG=${1:-fin}
ADER_AB_LIB=$PWD/paper_1212_3585_b200/libader_b200_prev.so python tools/flux_ab.py save gpurun_out/fi_prev.npz > gpurun_out/fi_prev.log 2>&1 || tail gpurun_out/fi_prev.log
python tools/flux_ab.py save gpurun_out/fi_new.npz > gpurun_out/fi_new.log 2>&1 || tail gpurun_out/fi_new.log
python tools/flux_ab.py cmp gpurun_out/fi_prev.npz gpurun_out/fi_new.npz | tee gpurun_out/flux_interior_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/fi_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"; }
L=paper_1212_3585_b200/libader_b200.so
cp $L /tmp/ader_new.so
for lib in prev new prev new; do
  if [ $lib = prev ]; then cp paper_1212_3585_b200/libader_b200_prev.so $L; else cp /tmp/ader_new.so $L; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c4_$lib.log 2>&1; show gpurun_out/b_${TAG}_c4_$lib.log "$lib c4"
done
cp /tmp/ader_new.so $L
