#!/bin/bash
# round-2 evidence: bench lines of every config, launch list + ncu --set full of
# timed-window steps (C4 step 5 of --steps 3 --warmup 3; C2 step 5), C2 with the R25 guess
mkdir -p gpurun_out
TAG=${1:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_${TAG}_$name.log 2>gpurun_out/bench_${TAG}_$name.err; echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_$name.log | cut -c1-200; }
run c4 ; run c4b ; run c2 --config c2 --n 512 ; run c2guess --config c2 --n 512 --pred-guess 1 --no-cpu-baseline
run c3 --config c3 ; run c5 --config c5 ; run c4osher --n 128 --flux osher ; run c6 --config c6 --steps 5 --no-cpu-baseline
run c1 --config c1 --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_reference.log 2>&1; echo "reference rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux|k_weno|k_update" -s 24 -c 6 -o gpurun_out/prof_${TAG}_c4_step5 $CMD > gpurun_out/ncu_${TAG}_c4.log 2>&1; echo "ncu c4 rc=$?"
CMD2="python bench.py --config c2 --n 512 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predictor|k_face_flux|k_weno|k_update" -s 20 -c 5 -o gpurun_out/prof_${TAG}_c2_step5 $CMD2 > gpurun_out/ncu_${TAG}_c2.log 2>&1; echo "ncu c2 rc=$?"
