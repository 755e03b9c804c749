#!/bin/bash
# per-kernel registers / spills of a .cu file for sm_100a: tools/regs.sh file.cu [regex]
cd "$(dirname "$1")"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include --expt-relaxed-constexpr \
  -Xptxas -v -diag-suppress 177 -c "$(basename "$1")" -o /tmp/regs_probe.o 2>&1 | python3 -c '
import re, sys
fn = None
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    m = re.search(r"(?:Compiling entry function|Function properties for) .(\S+).", line)
    if m: fn = m.group(1)
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and fn: spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and fn and re.search(pat, fn):
        print(m.group(1), "regs", "spill", spill, fn[:110])
' "${2:-}"
