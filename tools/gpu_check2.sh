#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED|^E   .*(assert|Error)" gpurun_out/pytest_gpu.log | grep -v "where\|+" | head -40
timeout 900 python tools/explosion_probe.py oracle > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe.log | cut -c1-300
