"""Full-time AMR runs: BASELINE C3 / C5 at full size on the GPU (completion,
steps, cell counts, conservation), and downscaled full-time twins against the
AMR oracle (cell sets bit-exact, active averages within the 1e-8 bar).
Prints one JSON line per run; used for profiles/round1_amr_full_runs.jsonl."""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def solver(wl, n=None):
    n = n or wl.n
    cfg = ader.make_config(dim=wl.dim, degree=wl.degree, n0=n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                           gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, lmax=wl.lmax, refine_factor=wl.refine_factor,
                           chi_ref=wl.chi_ref, chi_rec=wl.chi_rec, adapt_every=1, device=0)
    s = ader.Solver(cfg)
    s.set_initial(wl.ic)
    return s


def cells(s):
    arr = s.get_cells()
    lv = np.array([c.level for c in arr])
    st = np.array([c.status for c in arr])
    ix = np.array([list(c.idx) for c in arr]).reshape(-1, 3)
    u = np.array([list(c.u)[:s.nv] for c in arr]).reshape(-1, s.nv)
    return lv, st, ix, u


def totals(lv, st, u, wl, n):
    vol0 = np.prod([(wl.hi[k] - wl.lo[k]) / n[k] for k in range(wl.dim)])
    vol = vol0 / (wl.refine_factor ** wl.dim) ** lv
    a = st == 0
    return (u[a] * vol[a, None]).sum(0)


def full(name):
    wl = W.config(name)
    s = solver(wl)
    lv, st, ix, u = cells(s)
    t0 = totals(lv, st, u, wl, wl.n)
    w0 = time.time()
    try:
        r = s.step(wl.t_end, 10 ** 6)
        ok, err = True, ""
    except ader.AderError as e:
        ok, err, r = False, str(e), None
    lv, st, ix, u = cells(s)
    t1 = totals(lv, st, u, wl, wl.n)
    out = dict(run=f"{name}_full_gpu", ok=ok, err=err, t=s.t, wall_s=time.time() - w0,
               macro_steps=(r.macro_steps if r else None), cell_updates=(r.cell_updates if r else None),
               active_per_level=[int(((lv == l) & (st == 0)).sum()) for l in range(wl.lmax + 1)],
               mass_drift_rel=float(abs(t1[0] - t0[0]) / abs(t0[0])))
    print(json.dumps(out), flush=True)


def twin(name, n, lmax, t_end=None):
    import oracle as O
    wl = W.config(name)
    wl.lmax = lmax
    t_end = t_end if t_end is not None else wl.t_end
    s = solver(wl, n)
    o = O.AmrOracle(dim=wl.dim, degree=wl.degree, n=n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                    gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, lmax=lmax, refine_factor=wl.refine_factor,
                    chi_ref=wl.chi_ref, chi_rec=wl.chi_rec)
    o.set_initial(wl.ic)
    w0 = time.time()
    rg = s.step(t_end, 10 ** 6)
    w1 = time.time()
    ro = o.step(t_end, 10 ** 6)
    w2 = time.time()
    lg, sg, ig, ug = cells(s)
    lo_, so, io, uo = o.cells()
    same = len(lg) == len(lo_) and np.array_equal(lg, lo_) and np.array_equal(ig, io) and np.array_equal(sg, so)
    err = None
    if same:
        a = so == 0
        scale = np.maximum(np.abs(uo[a]).max(axis=0), np.abs(uo[a, 0]).max())
        err = float((np.abs(ug[a] - uo[a]).max(axis=0) / scale).max())
    out = dict(run=f"{name}_twin_{n[0]}_l{lmax}_t{t_end}", cell_sets_identical=bool(same), max_rel_err=err,
               gpu_steps=rg.macro_steps, oracle_steps=ro.steps, gpu_updates=rg.cell_updates,
               oracle_updates=ro.cell_updates, gpu_wall_s=w1 - w0, oracle_wall_s=w2 - w1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["full"]
    if "full" in which:
        full("c3")
        full("c5")
    if "twins" in which:
        twin("c3", (24, 24), 2)
        twin("c5", (24, 24), 2, 0.5)
