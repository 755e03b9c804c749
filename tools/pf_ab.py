"""A/B check of the fused predictor + face-flux walk (pred_flux.cu) against the
separate kernels on the GPU: the FLUX stage dump and the state after a few
steps must be bitwise equal (same arithmetic in the same order).

  python tools/pf_ab.py            (prints one line per array, exit 1 on a difference)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402

E3 = dict(dim=3, degree=2, lo=(-1,) * 3, hi=(1,) * 3)
CASES = {
    "c4_expl3d_24": (dict(E3, n0=(24, 20, 22), bc=(1,) * 6, cfl=0.3), lambda: W.explosion(3), 3),
    "expl3d_walls": (dict(E3, n0=(13, 11, 9), bc=(2, 1, 1, 2, 2, 1), cfl=0.3), lambda: W.explosion(3), 2),
    "expl3d_periodic_tall": (dict(E3, n0=(9, 7, 40), bc=(0,) * 6, cfl=0.3), lambda: W.explosion(3), 2),
    "osher3d": (dict(E3, n0=(14, 12, 10), bc=(1,) * 6, cfl=0.3, flux=1), lambda: W.explosion(3), 2),
    "mhd3d": (dict(dim=3, degree=2, n0=(9, 10, 11), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6, system=ader.MHD_GLM,
                   gamma=5 / 3, ch=2.0, cfl=0.3), lambda: W.random_smooth(3, system=1, amp=0.05), 2),
    "entropy3d_exact": (dict(dim=3, degree=2, n0=(10, 9, 8), lo=(0,) * 3, hi=(1,) * 3, bc=(4,) * 6, cfl=0.3,
                             exact_vel=(0.8, 0.35, -0.2)), lambda: W.entropy_wave(3, amp=0.2, v=(0.8, 0.35, -0.2)), 3),
    "vortex_m3": (dict(dim=2, degree=3, n0=(37, 29), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                  lambda: W.isentropic_vortex(), 3),
    "vortex_m2": (dict(dim=2, degree=2, n0=(33, 31), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                  lambda: W.isentropic_vortex(), 3),
    "expl2d_walls_m3": (dict(dim=2, degree=3, n0=(30, 26), lo=(-1, -1), hi=(1, 1), bc=(2, 1, 1, 2), cfl=0.45),
                        lambda: W.explosion(2), 3),
    "ot_m3": (dict(dim=2, degree=3, n0=(21, 19), lo=(0, 0), hi=(2 * np.pi, 2 * np.pi), bc=(0,) * 6,
                   system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.5), lambda: W.orszag_tang(), 2),
    "ot_m2": (dict(dim=2, degree=2, n0=(22, 18), lo=(0, 0), hi=(2 * np.pi, 2 * np.pi), bc=(0,) * 6,
                   system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.5), lambda: W.orszag_tang(), 2),
    "dmr2": (dict(dim=2, degree=2, n0=(60, 20), lo=(0, 0), hi=(3, 1), bc=(4, 4, 2, 4, 0, 0), cfl=0.45,
                  exact_vel=W.dmr_front_vel(2.0)), lambda: W.double_mach_reflection(2.0), 4),
    "expl2d_inflow": (dict(dim=2, degree=2, n0=(26, 21), lo=(-1, -1), hi=(1, 1), bc=(3, 3, 1, 1), cfl=0.45),
                      lambda: W.explosion(2), 3),
}


def run(sep):
    out = {}
    for name, (cfg, ic, steps) in CASES.items():
        s = ader.Solver(ader.make_config(device=0, fuse_pred_flux=1 - sep, **cfg))
        s.set_initial(ic())
        out[name + "_F"] = s.debug_dump(2, dt=1e-3)
        s.step(1e300, steps)
        out[name + "_u"] = s.get_state()
        s.close()
    return out


if __name__ == "__main__":
    A, B = run(1), run(0)
    bad = 0
    for k in A:
        same = np.array_equal(A[k], B[k])
        d = np.abs(A[k] - B[k]).max()
        print(f"{k:28s} bitwise={same} maxdiff={d:.3e}")
        bad += not same
    print("ALL BITWISE EQUAL" if bad == 0 else f"{bad} DIFFER")
    sys.exit(1 if bad else 0)
