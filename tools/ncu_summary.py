"""Summarise an ncu report: per kernel duration, DRAM bytes, FP64 pipe, occupancy,
issue, top SASS opcodes and top stall lines.  usage: ncu_summary.py rep [--sass]"""
import collections
import csv
import subprocess
import sys


def raw(rep):
    t = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(t.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    h, u, rows = raw(rep)
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
            "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "sm__maximum_warps_per_active_cycle_pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
    for r in rows:
        print("--")
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"  {w:60s} {r[i]} {u[i]}")
    if "--sass" in sys.argv:
        t = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                           capture_output=True, text=True).stdout
        blocks = t.split('"Kernel Name"')
        for b in blocks[1:]:
            rr = list(csv.reader(b.splitlines()))
            name = rr[0][1][:60] if len(rr[0]) > 1 else "?"
            hdr = rr[1]
            si, ni, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
            ops, st = collections.Counter(), collections.Counter()
            ti = ts = 0
            for r in rr[2:]:
                try:
                    s, i = int(r[ni]), int(r[ie])
                except (ValueError, IndexError):
                    continue
                src = r[si].strip()
                tok = src.split()
                op = tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")
                op = op.split(".")[0]
                ops[op] += i; st[op] += s; ti += i; ts += s
            print(f"== {name}: {ti:.3e} inst")
            for op, i in ops.most_common(12):
                print(f"   {op:8s} inst {100*i/max(1,ti):5.1f}%  stall {100*st[op]/max(1,ts):5.1f}%")


if __name__ == "__main__":
    main()
