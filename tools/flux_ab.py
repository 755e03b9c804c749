"""A/B check of the face-flux kernels on the GPU: dump F (ader_debug_dump FLUX)
and the state after a few steps for several configurations, save them to an
npz; run once with ADER_FLUX_LEGACY=1 and once without, then compare bitwise.

  python tools/flux_ab.py save out.npz     (env selects the kernel)
  python tools/flux_ab.py cmp a.npz b.npz
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402

if __import__("os").environ.get("ADER_AB_LIB"):   # A/B against another build of the library
    ader.LIB_PATH = __import__("os").environ["ADER_AB_LIB"]

CASES = {
    "c4_expl3d_24": dict(cfg=dict(dim=3, degree=2, n0=(24, 20, 22), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, cfl=0.3),
                         ic=lambda: W.explosion(3), steps=3),
    "expl3d_walls": dict(cfg=dict(dim=3, degree=2, n0=(13, 11, 9), lo=(-1,) * 3, hi=(1,) * 3, bc=(2, 1, 1, 2, 2, 1),
                                  cfl=0.3), ic=lambda: W.explosion(3), steps=2),
    "vortex_m3": dict(cfg=dict(dim=2, degree=3, n0=(37, 29), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                      ic=lambda: W.isentropic_vortex(), steps=3),
    "vortex_m2": dict(cfg=dict(dim=2, degree=2, n0=(33, 31), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                      ic=lambda: W.isentropic_vortex(), steps=3),
    "ot_m3": dict(cfg=dict(dim=2, degree=3, n0=(21, 19), lo=(0, 0), hi=(2 * np.pi, 2 * np.pi), bc=(0,) * 6,
                           system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.5), ic=lambda: W.orszag_tang(), steps=2),
    "mhd3d": dict(cfg=dict(dim=3, degree=2, n0=(9, 10, 11), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6,
                           system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.3),
                  ic=lambda: W.random_smooth(3, system=1, amp=0.05), steps=2),
    "osher3d": dict(cfg=dict(dim=3, degree=2, n0=(14, 12, 10), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, cfl=0.3,
                             flux=1), ic=lambda: W.explosion(3), steps=2),
}


def save(path):
    out = {}
    for name, c in CASES.items():
        s = ader.Solver(ader.make_config(device=0, **c["cfg"]))
        s.set_initial(c["ic"]())
        out[name + "_F"] = s.debug_dump(2, dt=1e-3)
        out[name + "_q"] = s.debug_dump(1, dt=1e-3)
        rep = s.step(1e300, c["steps"])
        out[name + "_u"] = s.get_state()
        out[name + "_flatcount"] = np.array([rep.pred_flat_cells, rep.pred_cells], dtype=float)
        s.close()
    np.savez(path, **out)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        if k.endswith("_flatcount"):
            print(f"{k:20s} flat/predicted cells {A[k].tolist()} vs {B[k].tolist()}")
            continue
        same = np.array_equal(A[k], B[k])
        d = np.abs(A[k] - B[k]).max()
        rel = d / max(np.abs(A[k]).max(), 1e-300)
        print(f"{k:20s} bitwise={same} maxdiff={d:.3e} rel={rel:.3e}")
        bad += rel > 1e-13
    print("ALL WITHIN 1e-13 (max-norm relative)" if bad == 0 else f"{bad} DIFFER")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2])
    else:
        sys.exit(1 if cmp(sys.argv[2], sys.argv[3]) else 0)
