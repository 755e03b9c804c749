#!/bin/bash
# multi-rank AMR compute sets (R28): loopback bitwise tests + computed/owned ratios
mkdir -p gpurun_out
TAG=${1:-rs}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_amr.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_$TAG.log | head -10
timeout 1200 python tools/amr_rank_sets.py --w 8 --steps 3 c3 > gpurun_out/ranksets_$TAG.jsonl 2>&1; echo "c3 rc=$?"
timeout 1200 python tools/amr_rank_sets.py --w 8 --steps 2 --n 60 c5 >> gpurun_out/ranksets_$TAG.jsonl 2>&1; echo "c5 rc=$?"
timeout 1500 python tools/amr_rank_sets.py --w 8 --steps 2 --n 18 c6 >> gpurun_out/ranksets_$TAG.jsonl 2>&1; echo "c6 rc=$?"
cat gpurun_out/ranksets_$TAG.jsonl | tail -8
