"""Probe: 2D explosion (BASELINE config 3 physics) admissibility vs CFL on the
uniform fine grid (GPU) and on the AMR hierarchy (GPU)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def run(n, cfl, steps, lmax):
    wl = W.config("c3", n)
    cfg = ader.make_config(dim=2, degree=2, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=cfl, lmax=lmax,
                           refine_factor=3, adapt_every=1, device=0)
    s = ader.Solver(cfg)
    s.set_initial(wl.ic)
    try:
        r = s.step(1e300, steps)
        out = dict(n=n, lmax=lmax, cfl=cfl, ok=True, steps=r.macro_steps, t=r.t, updates=r.cell_updates,
                   sweeps=r.pred_sweeps_total / max(1, r.pred_cells), sweeps_max=r.pred_sweeps_max, wall=r.wall_s)
    except ader.AderError as e:
        out = dict(n=n, lmax=lmax, cfl=cfl, ok=False, err=str(e))
    s.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for cfl in (0.45, 0.3, 0.2):
        run(300, cfl, 20, 0)
        run(900, cfl, 20, 0)
        run(100, cfl, 5, 2)
