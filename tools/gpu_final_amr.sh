# final refresh after host-side AMR changes: full GPU suite, smoke, AMR bench lines
TAG=${1:-final2}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -1 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_${TAG}_$name.log 2>&1; echo "bench $name rc=$?"; grep '^{' gpurun_out/bench_${TAG}_$name.log | tail -1 | cut -c1-200; }
run c3 --config c3 ; run c5 --config c5 ; run c6 --config c6 --steps 5 --no-cpu-baseline
