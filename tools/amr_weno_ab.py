"""A/B check of the AMR reconstruction (ADER_AMR_WENO_PATCH=0: every cell from its own box; default: sibling
patches): cell sets and averages after a few macro steps for 2D M = 2 / M = 3 (Euler, MHD) and 3D trees,
saved to an npz; compare two files bitwise.

  python tools/amr_weno_ab.py save out.npz
  python tools/amr_weno_ab.py cmp a.npz b.npz
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402

if __import__("os").environ.get("ADER_AB_LIB"):   # A/B against another build of the library
    ader.LIB_PATH = __import__("os").environ["ADER_AB_LIB"]

TWO_PI = 2 * np.pi
CASES = {
    "expl2d_m2_l2": dict(cfg=dict(dim=2, degree=2, n0=(30, 30), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, cfl=0.45, lmax=2,
                                  refine_factor=3, adapt_every=1, chi_ref=0.1, chi_rec=0.05),
                         ic=lambda: W.explosion(2), steps=4),
    "expl2d_m2_walls": dict(cfg=dict(dim=2, degree=2, n0=(20, 16), lo=(0, 0), hi=(1, 1), bc=(2, 1, 2, 1, 1, 1),
                                     cfl=0.45, lmax=2, refine_factor=3, adapt_every=1, chi_ref=0.1, chi_rec=0.05),
                            ic=lambda: W.explosion(2), steps=3),
    "expl2d_m3_l1": dict(cfg=dict(dim=2, degree=3, n0=(18, 18), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, cfl=0.45,
                                  lmax=1, refine_factor=3, adapt_every=1), ic=lambda: W.explosion(2), steps=2),
    "ot_m3_l2": dict(cfg=dict(dim=2, degree=3, n0=(16, 16), lo=(0, 0), hi=(TWO_PI, TWO_PI), bc=(0,) * 6,
                              system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.4, lmax=2, refine_factor=3,
                              adapt_every=1, chi_ref=0.05, chi_rec=0.02), ic=lambda: W.orszag_tang(), steps=3),
    "expl3d_l2": dict(cfg=dict(dim=3, degree=2, n0=(8, 8, 8), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, cfl=0.2,
                               lmax=2, refine_factor=3, adapt_every=1, chi_ref=0.05, chi_rec=0.025),
                      ic=lambda: W.explosion(3), steps=2),
}


def save(path):
    out = {}
    for name, c in CASES.items():
        s = ader.Solver(ader.make_config(device=0, **c["cfg"]))
        s.set_initial(c["ic"]())
        rep = s.step(1e300, c["steps"])
        cells = np.array([[x.level, x.status, *x.idx, *x.u] for x in s.get_cells()], dtype=float)
        out[name + "_cells"] = cells
        out[name + "_upd"] = np.array(list(rep.updates_per_level)[:4], dtype=float)
        print(name, "cells", cells.shape[0], "levels", np.bincount(cells[:, 0].astype(int)), flush=True)
        s.close()
    np.savez(path, **out)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        same = A[k].shape == B[k].shape and np.array_equal(A[k], B[k])
        print(f"{k:24s} bitwise={same}")
        bad += not same
    print("ALL BITWISE EQUAL" if bad == 0 else f"{bad} DIFFER")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2])
    else:
        sys.exit(1 if cmp(sys.argv[2], sys.argv[3]) else 0)
