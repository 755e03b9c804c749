#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_multirank.log 2>&1; echo "pytest multirank rc=$?"; tail -3 gpurun_out/pytest_multirank.log
grep -E "^FAILED|^E  " gpurun_out/pytest_multirank.log | head -10
timeout 1800 python tools/osher_probe.py > gpurun_out/osher_probe.jsonl 2> gpurun_out/osher_probe.err; echo "probe rc=$?"; cat gpurun_out/osher_probe.jsonl
