"""GPU parity on the configurations the round-1 review found untested
(north_star bar: <= 1e-8 after 100 steps; cell sets bit-exact; L1 against the
exact solution within 1 % of the oracle's).

Error scale (per variable): max_c |u_oracle[c, v]|; only a
variable that is zero in exact arithmetic (max below 1e-9 of the density
scale) is measured against the density scale.  Long oracle runs use the
multi-process runner (tests/parallel_oracle.py, bitwise the serial oracle)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import ader
from paper_1212_3585_b200 import workloads as W
from tests import parallel_oracle as PO

pytestmark = pytest.mark.gpu


def rel_err_v(a, b):
    b2 = b.reshape(-1, b.shape[-1])
    a2 = a.reshape(-1, a.shape[-1])
    sv = np.abs(b2).max(axis=0)
    rho = np.abs(b2[:, 0]).max()
    scale = np.where(sv > 1e-6 * rho, sv, rho)
    return (np.abs(a2 - b2).max(axis=0) / scale).max()


def gpu_run(kw, ic, t_end=1e300, steps=1):
    cfg = ader.make_config(device=0, n0=kw["n"], **{k: v for k, v in kw.items() if k != "n"})
    g = ader.Solver(cfg)
    g.set_initial(ic)
    rep = g.step(t_end, steps)
    u = g.get_state()
    g.close()
    return u, rep


CASES_100 = {
    # 2D vortex at order 4 (BASELINE configs[1] scheme), 100 steps
    "vortex2d_M3_24": (dict(dim=2, degree=3, n=(24, 24), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                       W.isentropic_vortex()),
    # Orszag-Tang at order 4 (BASELINE configs[4] physics), 16^2, 100 steps to
    # t = 2.69 (at CFL 0.9 the coarse 16^2 run reaches an inadmissible state by
    # t = 2.6, step ~32; CFL 0.3 runs the 100 steps in the oracle and on the GPU)
    "orszag_tang_M3_16": (dict(dim=2, degree=3, n=(16, 16), lo=(0, 0), hi=(2 * math.pi, 2 * math.pi),
                               bc=(0,) * 6, system=ader.MHD_GLM, gamma=5 / 3, ch=2.0, cfl=0.3), W.orszag_tang()),
    # 3D explosion at the C4 CFL (reading R1), 16^3, 100 steps
    "explosion3d_16": (dict(dim=3, degree=2, n=(16, 16, 16), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, cfl=0.3),
                       W.explosion(3)),
    # 3D random smooth periodic state, 12^3, 100 steps
    "random3d_periodic_12": (dict(dim=3, degree=2, n=(12, 12, 12), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6, cfl=0.9),
                             W.random_smooth(3, seed=1212, amp=0.08)),
}


@pytest.mark.parametrize("name", list(CASES_100))
def test_100_steps(name):
    kw, ic = CASES_100[name]
    ug, rep = gpu_run(kw, ic, steps=100)
    uo, steps, t = PO.run(kw, ic, max_steps=100)
    assert rep.macro_steps == steps == 100
    assert abs(rep.t - t) <= 1e-10 * t   # 100 CFL time steps from states equal to ~1e-12
    err = rel_err_v(ug, uo)
    assert err <= 1e-8, err
    if all(b == 0 for b in kw["bc"]):   # periodic: totals conserved to round-off
        u0, _ = gpu_run(kw, ic, steps=0)
        # (variables with zero total, e.g. psi of Orszag-Tang, against the mass scale)
        scale = np.maximum(np.abs(u0).sum(0), np.abs(u0[:, 0]).sum())
        assert np.all(np.abs(ug.sum(0) - u0.sum(0)) <= 1e-11 * scale)


def test_c2_l1_error_within_one_percent_of_the_oracle():
    # BASELINE configs[1] at 64^2 to t = 2 (77 steps): L1 of rho against the
    # exact (advected) vortex, GPU vs oracle
    t_end = 2.0
    kw = dict(dim=2, degree=3, n=(64, 64), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9)
    ug, rep = gpu_run(kw, W.isentropic_vortex(), t_end=t_end, steps=10 ** 6)
    uo, steps, t = PO.run(kw, W.isentropic_vortex(), t_end=t_end, max_steps=10 ** 6)
    assert rep.macro_steps == steps and abs(rep.t - t_end) < 1e-12
    ex = O.Oracle(dim=2, degree=3, n=(64, 64), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, ic_quad=6)
    ex.set_initial(W.vortex_exact(t_end))
    ue = ex.get_cells()
    l1g = np.abs(ug[:, 0] - ue[:, 0]).mean()
    l1o = np.abs(uo[:, 0] - ue[:, 0]).mean()
    assert abs(l1g - l1o) <= 0.01 * l1o, (l1g, l1o)
    assert rel_err_v(ug, uo) <= 1e-8


# ---------------------------------------------------------------------------
# AMR: populated lmax = 3 (Euler, MHD) and a 3D lmax = 2 twin
# ---------------------------------------------------------------------------

def gpu_cells(s):
    arr = s.get_cells()
    lv = np.array([c.level for c in arr], dtype=np.int32)
    st = np.array([c.status for c in arr], dtype=np.int32)
    ix = np.array([list(c.idx) for c in arr], dtype=np.int64).reshape(-1, 3)
    u = np.array([list(c.u)[:s.nv] for c in arr]).reshape(-1, s.nv)
    return lv, st, ix, u


def mhd_blast(radius=0.15):
    # magnetised blast: (rho, p) = (1, 1) inside r < radius, (0.5, 0.5) outside,
    # uniform B = sqrt(4 pi) (0.3, 0.2, 0) (Gaussian units)
    s = math.sqrt(4 * math.pi)

    def ic(x):
        out = np.zeros((x.shape[0], 9))
        inner = x[:, 0] ** 2 + x[:, 1] ** 2 < radius ** 2
        out[:, 0] = np.where(inner, 1.0, 0.5)
        out[:, 4] = np.where(inner, 1.0, 0.5)
        out[:, 5] = 0.3 * s
        out[:, 6] = 0.2 * s
        return out
    return ic


AMR = {
    "euler2d_lmax3": (dict(dim=2, degree=2, n=(6, 6), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=3, cfl=0.45,
                           chi_ref=0.1, chi_rec=0.05), W.explosion(2, radius=0.15), 4),
    "mhd2d_lmax3": (dict(dim=2, degree=2, n=(6, 6), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=3, cfl=0.4,
                         chi_ref=0.05, chi_rec=0.025, system=ader.MHD_GLM, gamma=5 / 3, ch=2.0), mhd_blast(), 4),
    # (the AMR oracle needs ~3 min for these 2 macro steps: 1e5 level-2 updates)
    "euler3d_lmax2_6": (dict(dim=3, degree=2, n=(6, 6, 6), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, lmax=2, cfl=0.2,
                             chi_ref=0.1, chi_rec=0.05), W.explosion(3, radius=0.2), 2),
}


@pytest.mark.parametrize("name", list(AMR))
def test_amr_deep_levels(name):
    kw, ic, steps = AMR[name]
    cfg = ader.make_config(device=0, n0=kw["n"], refine_factor=3, adapt_every=1,
                           **{k: v for k, v in kw.items() if k != "n"})
    g = ader.Solver(cfg)
    g.set_initial(ic)
    o = O.AmrOracle(refine_factor=3, **kw)
    o.set_initial(ic)
    for _ in range(steps):
        rg = g.step(1e300, 1)
        ro = o.step(1e300, 1)
        assert list(rg.updates_per_level) == list(ro.updates_per_level)
        assert ro.min_threshold_margin > 1e-8 and rg.min_threshold_margin > 1e-8
        assert abs(rg.min_threshold_margin - ro.min_threshold_margin) <= 1e-6 * max(1.0, ro.min_threshold_margin)
    lg, sg, ig, ug = gpu_cells(g)
    lo_, so, io, uo = o.cells()
    assert np.array_equal(lg, lo_) and np.array_equal(ig, io) and np.array_equal(sg, so)
    for l in range(2, kw["lmax"] + 1):   # the deep levels are populated
        assert ((lo_ == l) & (so == 0)).sum() > 0, l
    act = so == 0
    err = rel_err_v(ug[act], uo[act])
    assert err <= 1e-9, err


# ---------------------------------------------------------------------------
# predictor initial guess (reading R25), GPU vs oracle
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kw,ic", [
    (dict(dim=2, degree=3, n=(32, 32), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9), W.isentropic_vortex()),
    (dict(dim=3, degree=2, n=(10, 9, 8), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6, cfl=0.5),
     W.random_smooth(3, seed=3585, amp=0.08)),
])
def test_predictor_guess_parity_and_sweeps(kw, ic):
    res = {}
    for guess in (0, 1):
        cfg = ader.make_config(device=0, n0=kw["n"], pred_guess=guess, **{k: v for k, v in kw.items() if k != "n"})
        g = ader.Solver(cfg)
        g.set_initial(ic)
        g.step(1e300, 1)                      # the first step has no previous q (R3)
        rep = g.step(1e300, 4)
        res[guess] = (g.get_state(), rep.pred_sweeps_total / rep.pred_cells)
        g.close()
        o = O.Oracle(pred_guess=guess, **kw)
        o.set_initial(ic)
        o.step(1e300, 1)
        o.step(1e300, 4)
        assert rel_err_v(res[guess][0], o.get_cells()) <= 1e-10
    # the converged predictor differs only within its tolerance (R2)
    assert rel_err_v(res[1][0], res[0][0]) <= 1e-11
    assert res[1][1] < res[0][1], (res[1][1], res[0][1])



# ---------------------------------------------------------------------------
# time-dependent exact boundaries (reading R26), GPU vs oracle
# ---------------------------------------------------------------------------

EXACT_CASES = {
    "traveling2d_M2": (dict(dim=2, degree=2, n=(20, 18), lo=(0, 0), hi=(1, 1), bc=(4,) * 6, cfl=0.9,
                            exact_vel=(0.8, 0.35, 0.0)), W.entropy_wave(2, amp=0.2, v=(0.8, 0.35, 0.0)), 25),
    "traveling2d_M3": (dict(dim=2, degree=3, n=(16, 15), lo=(0, 0), hi=(1, 1), bc=(4,) * 6, cfl=0.9,
                            exact_vel=(0.8, 0.35, 0.0)), W.entropy_wave(2, amp=0.2, v=(0.8, 0.35, 0.0)), 25),
    "traveling3d_M2": (dict(dim=3, degree=2, n=(10, 9, 8), lo=(0,) * 3, hi=(1,) * 3, bc=(4,) * 6, cfl=0.5,
                            exact_vel=(0.8, 0.35, -0.2)), W.entropy_wave(3, amp=0.2, v=(0.8, 0.35, -0.2)), 10),
    # the double Mach reflection geometry at shock Mach 2 (reading R27)
    "dmr2_60x20": (dict(dim=2, degree=2, n=(60, 20), lo=(0, 0), hi=(3, 1), bc=(4, 4, 2, 4, 0, 0), cfl=0.45,
                        exact_vel=W.dmr_front_vel(2.0)), W.double_mach_reflection(2.0), 60),
}


@pytest.mark.parametrize("name", list(EXACT_CASES))
def test_exact_boundary_parity(name):
    kw, ic, steps = EXACT_CASES[name]
    ug, rep = gpu_run(kw, ic, steps=steps)
    o = O.Oracle(**kw)
    o.set_initial(ic)
    ro = o.step(1e300, steps)
    assert rep.macro_steps == ro.steps == steps
    err = rel_err_v(ug, o.get_cells())
    assert err <= 1e-9, err
