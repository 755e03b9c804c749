"""Full-time AMR run of a named workload on the GPU (default c6, the paper's 3D
AMR explosion to t = 0.25): macro steps, cell updates, final tree
size (the paper reports 9,079,984 elements at t = 0.25 for its run), wall time,
conservation drift.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def main(name="c6", t_end=None):
    wl = W.config(name)
    cfg = ader.make_config(dim=wl.dim, degree=wl.degree, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                           gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, lmax=wl.lmax, refine_factor=wl.refine_factor,
                           chi_ref=wl.chi_ref, chi_rec=wl.chi_rec, adapt_every=1, device=0)
    s = ader.Solver(cfg)
    t0 = time.time()
    s.set_initial(wl.ic)
    t_init = time.time() - t0
    n_init = len(s.get_cells())
    t_end = t_end or wl.t_end
    t0 = time.time()
    rep = s.step(t_end, 10 ** 6)
    wall = time.time() - t0
    cells = s.get_cells()
    lv = np.array([c.level for c in cells])
    st = np.array([c.status for c in cells])
    out = dict(workload=wl.name, t=rep.t, macro_steps=rep.macro_steps, cell_updates=rep.cell_updates,
               updates_per_level=list(rep.updates_per_level)[:wl.lmax + 1], wall_s=wall, init_s=t_init,
               cells_initial=n_init, cells_final=len(cells), active_final=int((st == 0).sum()),
               active_per_level=[int(((st == 0) & (lv == l)).sum()) for l in range(wl.lmax + 1)],
               cell_updates_per_s=rep.cell_updates / wall,
               paper_final_elements=9079984 if name == "c6" else None)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c6"]))
