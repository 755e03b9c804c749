"""Per-kernel DRAM bytes and hardware-counted FP64 rate from an ncu --set full
report -> profiles/ncu_traffic.json entry.  usage: ncu_to_json.py rep workload [flux] [source label]

fp64_hw_frac = (2 dfma + dadd + dmul thread instructions per cycle) / (2 x
peak dfma thread instructions per cycle), i.e. the FP64 pipe's flop rate as
counted by the hardware, next to the algorithmic rate bench.py
reports."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = [("k_predictor", "stdg_predictor"), ("k_face_flux", "face_flux_rusanov"), ("k_weno<2, 2", "weno_z_sweep"),
         ("k_update", "fv_update")]


def main(rep, workload, flux="rusanov", label=""):
    t = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(t.splitlines()))
    h, u = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}

    def val(r, k):
        x = float(r[col[k]].replace(",", ""))
        unit = u[col[k]]
        return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
    out = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        for pat, key in NAMES:
            key = key.replace("rusanov", flux)
            if pat in name:
                out[f"{key}_dram_bytes_per_launch"] = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
                f = (2 * val(r, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
                     + val(r, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
                     + val(r, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"))
                peak = 2 * val(r, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
                out[f"{key}_fp64_hw_frac"] = f / peak
                break
    out["source"] = f"ncu --set full capture {os.path.basename(rep)}" + (f": {label}" if label else "")
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[workload] = out
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
