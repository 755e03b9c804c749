#!/bin/bash
# multi-rank AMR rows of w/q for computed cells only: loopback + 2-process tests, memory report
mkdir -p gpurun_out
TAG=${1:-sl}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo build failed; tail gpurun_out/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_amr.py tests/test_gpu_host_comm.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
grep -E "^FAILED|^E  " gpurun_out/pytest_$TAG.log | head -10
ADER_AMR_MEM=1 timeout 1200 python tools/amr_rank_sets.py --w 8 --steps 2 --n 18 --no-one c6 > gpurun_out/slots_${TAG}_c6.jsonl 2> gpurun_out/slots_${TAG}_c6.err; echo "c6 rc=$?"
tail -2 gpurun_out/slots_${TAG}_c6.jsonl; grep "amr memory" gpurun_out/slots_${TAG}_c6.err | tail -9
