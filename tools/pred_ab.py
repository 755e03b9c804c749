"""A/B check of predictor kernel variants on the GPU (the environment selects the
variant, e.g. ADER_PRED_DMMA=0): dumps q (ader_debug_dump PRED), the state or
the AMR cell set after a few steps and the sweep counters for 2D M = 3
configurations (uniform Euler with and without the R25 guess, walls, MHD
Orszag-Tang, AMR Euler and MHD) into an npz; compare two files bitwise and
by max relative difference.

  python tools/pred_ab.py save out.npz
  python tools/pred_ab.py cmp a.npz b.npz
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402

TWO_PI = 2 * np.pi
CASES = {
    "vortex_37x29": dict(cfg=dict(dim=2, degree=3, n0=(37, 29), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                         ic=lambda: W.isentropic_vortex(), steps=5),
    "vortex_64_guess": dict(cfg=dict(dim=2, degree=3, n0=(64, 64), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9,
                                     pred_guess=1), ic=lambda: W.isentropic_vortex(), steps=6),
    "expl2d_walls": dict(cfg=dict(dim=2, degree=3, n0=(41, 23), lo=(-1, -1), hi=(1, 1), bc=(2, 1, 1, 2, 1, 1),
                                  cfl=0.5), ic=lambda: W.explosion(2), steps=4),
    "ot_m3": dict(cfg=dict(dim=2, degree=3, n0=(21, 19), lo=(0, 0), hi=(TWO_PI, TWO_PI), bc=(0,) * 6,
                           system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.5), ic=lambda: W.orszag_tang(), steps=3),
    "expl2d_m3_amr": dict(cfg=dict(dim=2, degree=3, n0=(18, 18), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, cfl=0.45,
                                   lmax=1, refine_factor=3, adapt_every=1), ic=lambda: W.explosion(2), steps=2,
                          amr=True),
    "ot_m3_amr": dict(cfg=dict(dim=2, degree=3, n0=(16, 16), lo=(0, 0), hi=(TWO_PI, TWO_PI), bc=(0,) * 6,
                               system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.4, lmax=1, refine_factor=3,
                               adapt_every=1, chi_ref=0.05, chi_rec=0.02), ic=lambda: W.orszag_tang(), steps=3,
                      amr=True),
}


def save(path):
    out = {}
    for name, c in CASES.items():
        s = ader.Solver(ader.make_config(device=0, **c["cfg"]))
        s.set_initial(c["ic"]())
        if not c.get("amr"):
            out[name + "_q"] = s.debug_dump(1, dt=1e-3)
        rep = s.step(1e300, c["steps"])
        out[name + "_sweeps"] = np.array([rep.pred_sweeps_total, rep.pred_sweeps_max, rep.pred_cells], dtype=float)
        if c.get("amr"):
            out[name + "_cells"] = np.array([[x.level, x.status, *x.idx, *x.u] for x in s.get_cells()], dtype=float)
        else:
            out[name + "_u"] = s.get_state()
        s.close()
    np.savez(path, **out)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    worst = 0.0
    for k in A.files:
        same = np.array_equal(A[k], B[k])
        if A[k].shape != B[k].shape:
            print(f"{k:24s} SHAPE {A[k].shape} vs {B[k].shape}")
            worst = np.inf
            continue
        d = np.abs(A[k] - B[k])
        sc = np.maximum(np.abs(A[k]).max(axis=0, keepdims=True) if A[k].ndim > 1 else np.abs(A[k]).max(), 1e-300)
        rel = (d / sc).max() if d.size else 0.0
        if not k.endswith("_sweeps"):
            worst = max(worst, rel)
        print(f"{k:24s} bitwise={same} max rel (per-column scale) {rel:.3e}")
    print(f"worst relative difference (excluding sweep counters) {worst:.3e}")
    return worst


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2])
    else:
        sys.exit(0 if cmp(sys.argv[2], sys.argv[3]) < 1e-12 else 1)
