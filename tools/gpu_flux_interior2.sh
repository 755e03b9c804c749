#!/bin/bash
# A/B of the interior fast path of k_face_flux_cells against the previous build, then the uniform suites
mkdir -p gpurun_out
TAG=${1:-fi2}
ADER_AB_LIB=$PWD/paper_1212_3585_b200/libader_b200_prev.so python tools/flux_ab.py save gpurun_out/fi_prev.npz > gpurun_out/fi_prev.log 2>&1 || tail gpurun_out/fi_prev.log
python tools/flux_ab.py save gpurun_out/fi_new.npz > gpurun_out/fi_new.log 2>&1 || tail gpurun_out/fi_new.log
python tools/flux_ab.py cmp gpurun_out/fi_prev.npz gpurun_out/fi_new.npz | tee gpurun_out/flux_interior2_cmp_$TAG.log | grep -v "bitwise=True"
rm -f gpurun_out/fi_*.npz
show() { tail -1 $1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step'],3), [(e['kernel'], round(e['frac'],3), round(e['ms_per_launch'],3)) for e in d['roofline_kernels']])"; }
L=paper_1212_3585_b200/libader_b200.so
cp $L /tmp/ader_new.so
for lib in prev new prev new; do
  if [ $lib = prev ]; then cp paper_1212_3585_b200/libader_b200_prev.so $L; else cp /tmp/ader_new.so $L; fi
  timeout 600 python bench.py --config c2 --n 512 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_c2_$lib.log 2>&1; show gpurun_out/b_${TAG}_c2_$lib.log "$lib c2"
  timeout 600 python bench.py --n 128 --flux osher --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${TAG}_osh_$lib.log 2>&1; show gpurun_out/b_${TAG}_osh_$lib.log "$lib osher128"
done
cp /tmp/ader_new.so $L
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c4.log 2>gpurun_out/bench_${TAG}_c4.err; show gpurun_out/bench_${TAG}_c4.log "final c4"
timeout 900 python bench.py --config c2 --n 512 > gpurun_out/bench_${TAG}_c2.log 2>gpurun_out/bench_${TAG}_c2.err; show gpurun_out/bench_${TAG}_c2.log "final c2"
timeout 900 python bench.py --n 128 --flux osher > gpurun_out/bench_${TAG}_c4osher.log 2>gpurun_out/bench_${TAG}_c4osher.err; show gpurun_out/bench_${TAG}_c4osher.log "final c4osher"
