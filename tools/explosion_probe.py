"""Probe: does the 3D explosion (BASELINE config 4) stay admissible at a given
grid / CFL on the GPU, and does the oracle agree on a small grid?  Prints JSON
lines; used to decide reading R1's CFL for 3D."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def run(n, cfl, steps):
    wl = W.config("c4", n)
    cfg = ader.make_config(dim=3, degree=2, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=cfl, device=0)
    s = ader.Solver(cfg)
    s.set_initial(wl.ic)
    t0 = time.time()
    try:
        r = s.step(1e300, steps)
        out = dict(n=n, cfl=cfl, ok=True, steps=r.macro_steps, t=r.t, sweeps=r.pred_sweeps_total / max(1, r.pred_cells),
                   sweeps_max=r.pred_sweeps_max)
    except ader.AderError as e:
        out = dict(n=n, cfl=cfl, ok=False, err=str(e))
    out["wall"] = time.time() - t0
    s.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for n in (32, 64, 128, 256):
        for cfl in (0.9, 0.6, 0.5, 0.3):
            run(n, cfl, 25 if n < 256 else 10)
    if len(sys.argv) > 1 and sys.argv[1] == "oracle":
        import oracle as O
        n = 24
        wl = W.config("c4", n)
        cfg = ader.make_config(dim=3, degree=2, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=0.9, device=0)
        g = ader.Solver(cfg)
        g.set_initial(wl.ic)
        o = O.Oracle(dim=3, degree=2, n=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=0.9)
        o.set_initial(wl.ic)
        for k in range(3):
            try:
                g.step(1e300, 1)
                o.step(1e300, 1)
            except Exception as e:
                print(json.dumps(dict(oracle_cmp=k, err=str(e))))
                break
            ug, uo = g.get_state(), o.get_cells()
            print(json.dumps(dict(oracle_cmp=k, maxdiff=float(np.abs(ug - uo).max()))), flush=True)
