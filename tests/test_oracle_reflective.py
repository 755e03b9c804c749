"""Pins of the oracle's reflective walls (reading R22: the
blast-wave / DMR boundary condition of P:965-966).

The mirrored polynomial is pinned by point evaluation; the wall as a whole by
the mirror symmetry of the explosion (the quadrant [0,1]^2 with walls at x=0
and y=0 must reproduce the [-1,1]^2 solution restricted to that quadrant), and
by exact conservation of mass and energy in a closed box (a wall only carries
pressure, so only the normal momentum changes).
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W

E, T, P, R = O.EULER, O.TRANSMISSIVE, O.PERIODIC, O.REFLECTIVE


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_reflected_polynomial_is_the_mirror_image(d, M):
    rng = np.random.default_rng(1212)
    N = M + 1
    nv = d + 2
    q = rng.standard_normal((nv, N ** (d + 1)))
    lib = O.lib()
    dp = C.POINTER(C.c_double)
    lib.orc_reflect_poly.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp]
    lib.orc_eval_st.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, C.c_double, dp]

    def ev(qq, xi, tau):
        out = np.zeros(nv)
        lib.orc_eval_st(d, M, nv, O._p(qq), O._p(np.ascontiguousarray(xi)), tau, O._p(out))
        return out
    for direction in range(d):
        out = np.zeros_like(q)
        lib.orc_reflect_poly(d, M, nv, direction, O._p(q), O._p(out))
        for _ in range(5):
            xi = rng.uniform(0, 1, 3)
            tau = rng.uniform()
            xm = xi.copy()
            xm[direction] = 1.0 - xi[direction]
            a = ev(out, xi, tau)
            b = ev(q, xm, tau)
            b[1 + direction] = -b[1 + direction]
            np.testing.assert_allclose(a, b, atol=1e-12)


def _pulse(x):
    # smooth pressure / density pulse centred at the origin: even in x and y
    r2 = x[:, 0] ** 2 + x[:, 1] ** 2
    out = np.zeros((x.shape[0], 9))
    out[:, 0] = 1.0 + 0.2 * np.exp(-10.0 * r2)
    out[:, 4] = 1.0 + 0.3 * np.exp(-10.0 * r2)
    return out


@pytest.mark.parametrize("M,m", [(2, 10), (3, 8)])
def test_explosion_quadrant_with_walls_matches_full_domain(M, m):
    full = O.Oracle(dim=2, degree=M, n=(2 * m, 2 * m), lo=(-1, -1), hi=(1, 1), bc=(T,) * 6, cfl=0.45)
    quad = O.Oracle(dim=2, degree=M, n=(m, m), lo=(0, 0), hi=(1, 1), bc=(R, T, R, T, 0, 0), cfl=0.45)
    ic = W.explosion(2) if M == 2 else _pulse
    full.set_initial(ic)
    quad.set_initial(ic)
    for _ in range(4):
        dt = full.compute_dt()
        assert abs(quad.compute_dt() - dt) <= 1e-13 * dt
        full.step(1e300, 1)
        quad.step(1e300, 1)
    uf = full.get_cells().reshape(2 * m, 2 * m, -1)[m:, m:]
    uq = quad.get_cells().reshape(m, m, -1)
    scale = np.abs(uf).reshape(-1, 4).max(0)
    scale = np.maximum(scale, scale[0])
    assert (np.abs(uq - uf).reshape(-1, 4).max(0) / scale).max() < 1e-11


def test_closed_box_conserves_mass_and_energy():
    for d, n in [(2, (10, 9)), (3, (6, 5, 7))]:
        o = O.Oracle(dim=d, degree=2, n=n, lo=(0,) * d, hi=(1,) * d, bc=(R,) * 6, cfl=0.45)
        o.set_initial(W.random_smooth(d, seed=1212, amp=0.2))
        u0 = o.get_cells()
        o.step(1e300, 5)
        u1 = o.get_cells()
        for v in (0, d + 1):
            assert abs(u1[:, v].sum() - u0[:, v].sum()) <= 1e-12 * np.abs(u0[:, v]).sum()
        assert not np.allclose(u1[:, 1], u0[:, 1], atol=1e-6)


def test_wall_at_rest_keeps_a_resting_gas():
    # gas at rest in a closed box stays at rest (the wall flux of a resting
    # state is pure pressure, (0, p, 0, 0)); the reflected trace is evaluated
    # with the mirrored basis, so the wall pressure agrees to round-off only
    o = O.Oracle(dim=2, degree=2, n=(7, 6), lo=(0, 0), hi=(1, 1), bc=(R,) * 6)
    o.set_initial(W.constant_state(rho=1.3, v=(0, 0, 0), p=0.7))
    u0 = o.get_cells()
    o.step(1e300, 3)
    np.testing.assert_allclose(o.get_cells(), u0, rtol=0, atol=1e-15)


def test_reflective_rejected_for_mhd_and_thin_axes():
    with pytest.raises(ValueError):
        O.Oracle(dim=2, system=O.MHD, degree=2, n=(8, 8), lo=(0, 0), hi=(1, 1), bc=(R, R, 0, 0, 0, 0))
    with pytest.raises(ValueError):
        O.Oracle(dim=2, degree=2, n=(2, 8), lo=(0, 0), hi=(1, 1), bc=(R, R, 0, 0, 0, 0))


def test_amr_closed_box_conserves_mass_and_energy():
    a = O.AmrOracle(dim=2, degree=2, n=(10, 10), lo=(0, 0), hi=(1, 1), bc=(R,) * 6, lmax=1, cfl=0.45,
                    chi_ref=0.02, chi_rec=0.01)
    a.set_initial(W.random_smooth(2, seed=3585, amp=0.25))

    def tot():
        lv, st, ix, u = a.cells()
        vol = np.array([(0.1 / 3 ** l) ** 2 for l in lv])
        act = st == 0
        return (u[act] * vol[act, None]).sum(0)
    t0 = tot()
    a.step(1e300, 3)
    t1 = tot()
    assert abs(t1[0] - t0[0]) <= 1e-13 * abs(t0[0]) and abs(t1[3] - t0[3]) <= 1e-13 * abs(t0[3])
