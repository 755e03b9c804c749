"""Pins of the oracle's physics, Rusanov flux, predictor and face quadrature
against closed forms and exactness properties (no GPU)."""
import math

import numpy as np
import pytest

import oracle as O

E, MHD = O.EULER, O.MHD


def test_euler_flux_free_stream():
    # eq:Euler-system @ P:838-867; (rho,v,p) = (1,(1,1,0),1) -> f = (1,2,1,0,4.5)
    u3 = O.prim_to_cons(E, 3, 1.4, [1, 1, 1, 0, 1])
    np.testing.assert_allclose(O.phys_flux(E, 3, 1.4, 0, u3, 0), [1, 2, 1, 0, 4.5], atol=1e-15)
    u2 = O.prim_to_cons(E, 2, 1.4, [1, 1, 1, 0, 1])
    np.testing.assert_allclose(u2, [1, 1, 1, 3.5], atol=1e-15)   # E = p/(g-1) + rho v^2/2
    np.testing.assert_allclose(O.phys_flux(E, 2, 1.4, 0, u2, 1), [1, 1, 2, 4.5], atol=1e-15)


def test_euler_sound_speed():
    u = O.prim_to_cons(E, 2, 1.4, [1, 0, 0, 0, 1])
    assert abs(O.max_speed(E, 2, 1.4, 0, u, 0) - math.sqrt(1.4)) < 1e-15
    u = O.prim_to_cons(E, 3, 1.4, [1, 3, 0, 0, 1 / 1.4])   # Mach-3 state: c = 1
    assert abs(O.max_speed(E, 3, 1.4, 0, u, 0) - 4.0) < 1e-14


def test_rusanov_sod_worked_example():
    # eqn.rusanov @ P:181-185 on Sod states (rho,v,p) = (1,0,1)|(0.125,0,0.1):
    # f_L = (0,1,0,0), f_R = (0,0.1,0,0), s_max = sqrt(1.4), u_R-u_L = (-0.875,0,0,-2.25)
    uL = O.prim_to_cons(E, 2, 1.4, [1, 0, 0, 0, 1])
    uR = O.prim_to_cons(E, 2, 1.4, [0.125, 0, 0, 0, 0.1])
    F = O.rusanov(E, 2, 1.4, 0, uL, uR, 0)
    s = math.sqrt(1.4)
    np.testing.assert_allclose(F, [0.5 * s * 0.875, 0.55, 0.0, 0.5 * s * 2.25], atol=1e-15)
    np.testing.assert_allclose(F, [0.5176569810212164, 0.55, 0, 1.3311179511974138], atol=1e-15)


def test_rusanov_consistency_and_mirror():
    rng = np.random.default_rng(1212)
    for _ in range(10):
        pr = [rng.uniform(0.5, 2), *rng.uniform(-1, 1, 3), rng.uniform(0.5, 2)]
        u = O.prim_to_cons(E, 3, 1.4, pr)
        for d in range(3):
            np.testing.assert_allclose(O.rusanov(E, 3, 1.4, 0, u, u, d), O.phys_flux(E, 3, 1.4, 0, u, d), atol=1e-14)
    # mirror symmetry: swapping states and reflecting the normal velocity flips the normal flux
    pl = [1.0, 0.3, 0.1, 0, 1.0]
    prr = [0.5, -0.2, 0.4, 0, 0.4]
    uL, uR = O.prim_to_cons(E, 2, 1.4, pl), O.prim_to_cons(E, 2, 1.4, prr)
    mL = O.prim_to_cons(E, 2, 1.4, [prr[0], -prr[1], prr[2], 0, prr[4]])
    mR = O.prim_to_cons(E, 2, 1.4, [pl[0], -pl[1], pl[2], 0, pl[4]])
    F = O.rusanov(E, 2, 1.4, 0, uL, uR, 0)
    G = O.rusanov(E, 2, 1.4, 0, mL, mR, 0)
    np.testing.assert_allclose(G, [-F[0], F[1], -F[2], -F[3]], atol=1e-14)


def test_mhd_flux_and_speed():
    # (rho,v,p,B,psi) = (1,0,1,(1,0,0),0), momentum-x row = 1 - 1/(8 pi)
    g, ch = 5 / 3, 2.0
    u = O.prim_to_cons(MHD, 2, g, [1, 0, 0, 0, 1, 1, 0, 0, 0])
    f = O.phys_flux(MHD, 2, g, ch, u, 0)
    assert abs(f[1] - (1 - 1 / (8 * math.pi))) < 1e-15
    assert f[0] == 0 and f[4] == 0 and abs(f[8] - ch * ch) < 1e-15
    # B = 0 reduces to the Euler sound speed (up to max with c_h)
    u = O.prim_to_cons(MHD, 2, g, [1, 0.1, 0, 0, 1, 0, 0, 0, 0])
    assert abs(O.max_speed(MHD, 2, g, 0.0, u, 0) - (0.1 + math.sqrt(g))) < 1e-14
    assert O.max_speed(MHD, 2, g, 5.0, u, 0) == 5.0
    # along B the fast speed is max(a, b_A); across B it is sqrt(a^2 + b^2)
    u = O.prim_to_cons(MHD, 2, g, [1, 0, 0, 0, 1, 3, 0, 0, 0])
    a2, b2 = g, 9 / (4 * math.pi)
    assert abs(O.max_speed(MHD, 2, g, 0, u, 0) - math.sqrt(max(a2, b2))) < 1e-14
    assert abs(O.max_speed(MHD, 2, g, 0, u, 1) - math.sqrt(a2 + b2)) < 1e-14


def _st_nodes(d, M):
    t = O.tables(M)
    N = M + 1
    idx = np.arange(N ** (d + 1))
    return t, [t["lam"][(idx // N ** k) % N] for k in range(d + 1)]


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_predictor_constant_state_fixed_point(d, M):
    nv = d + 2
    u = O.prim_to_cons(E, d, 1.4, [0.8, 0.3, -0.2, 0.1, 0.6])
    w = np.tile(u[:, None], (1, (M + 1) ** d))
    rc, q, sw = O.predict_cell(d, M, E, 1.4, 0, w, [0.3] * d)
    assert rc == 0 and sw <= 2
    np.testing.assert_allclose(q, np.tile(u[:, None], (1, (M + 1) ** (d + 1))), atol=1e-14)


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_predictor_exact_for_entropy_wave(d, M):
    # With v, p constant the Euler flux is linear in rho, so the weak problem
    # (eqn.pde.weak3 @ P:415-430) is solved exactly by rho(x - v t) when rho0
    # has total degree <= M; the Picard iteration is nilpotent for a linear
    # flux with index d*M+1, +1 sweep to detect convergence.
    t, X = _st_nodes(d, M)
    rng = np.random.default_rng(3585)
    v = np.array([0.7, -0.4, 0.25])[:d]
    p, g = 1.3, 1.4
    dtdx = np.array([0.35, 0.3, 0.25])[:d]
    # random polynomial of total degree M in d variables
    terms = [e for e in np.ndindex(*([M + 1] * d)) if sum(e) <= M]
    c = rng.normal(size=len(terms)) * 0.05

    def rho0(*xs):
        return 1.0 + sum(ci * np.prod([xs[k] ** e[k] for k in range(d)], axis=0) for ci, e in zip(c, terms))
    xs_sp = [X[k][: (M + 1) ** d] for k in range(d)]
    r0 = rho0(*xs_sp)
    nv = d + 2
    w = np.zeros((nv, (M + 1) ** d))
    w[0] = r0
    for k in range(d):
        w[1 + k] = r0 * v[k]
    w[1 + d] = p / (g - 1) + 0.5 * r0 * (v @ v)
    rc, q, sw = O.predict_cell(d, M, E, g, 0, w, dtdx, tol=1e-13, max_sweeps=40)
    assert rc == 0
    assert sw <= d * M + 2, sw
    tau = X[d]
    rex = rho0(*[X[k] - v[k] * dtdx[k] * tau for k in range(d)])
    np.testing.assert_allclose(q[0], rex, atol=1e-12)
    np.testing.assert_allclose(q[1 + d], p / (g - 1) + 0.5 * rex * (v @ v), atol=1e-12)


def test_predictor_nonconvergence_is_an_error():
    d, M = 2, 2
    u = O.prim_to_cons(E, d, 1.4, [1.0, 0.3, -0.2, 0, 0.6])
    rng = np.random.default_rng(1212)
    w = np.tile(u[:, None], (1, 9)) * (1 + 0.2 * rng.normal(size=(4, 9)))
    rc, q, sw = O.predict_cell(d, M, E, 1.4, 0, w, [0.4, 0.4], tol=1e-13, max_sweeps=2)
    assert rc == 3 and sw == 2


@pytest.mark.parametrize("d,M", [(2, 2), (3, 2), (2, 3)])
def test_face_flux_exact_for_continuous_linear_flux(d, M):
    # flux:F: if both sides trace the same polynomial the Rusanov
    # dissipation vanishes and the Gauss rule (exact to degree 2M+1) integrates
    # the linear flux exactly.  q_L, q_R: the entropy-wave polynomial with the
    # face at xi = 1 of L and xi = 0 of R.
    t, X = _st_nodes(d, M)
    v = np.array([0.7, -0.4, 0.25])[:d]
    p, g = 1.3, 1.4
    a = np.array([0.11, -0.07, 0.05])[:d]
    at = 0.03

    def rho(xs, tau):
        return 1.0 + sum(a[k] * xs[k] for k in range(d)) + at * tau
    nv = d + 2

    def cons(r):
        out = np.zeros((nv, r.size))
        out[0] = r
        for k in range(d):
            out[1 + k] = r * v[k]
        out[1 + d] = p / (g - 1) + 0.5 * r * (v @ v)
        return out
    tau = X[d]
    qL = cons(rho([X[k] - (1.0 if k == 0 else 0.0) for k in range(d)], tau))
    qR = cons(rho([X[k] for k in range(d)], tau))
    F = O.face_flux(d, M, E, g, 0, 0, qL, qR)
    # exact face-time average of rho over xi=0, eta,zeta,tau in [0,1]: 1 + sum_{k>0} a_k/2 + at/2
    rbar = 1.0 + sum(a[k] * 0.5 for k in range(1, d)) + at * 0.5
    ref = np.zeros(nv)
    ref[0] = rbar * v[0]
    for k in range(d):
        ref[1 + k] = rbar * v[0] * v[k] + (p if k == 0 else 0.0)
    ref[1 + d] = v[0] * (p / (g - 1) + 0.5 * rbar * (v @ v) + p)
    np.testing.assert_allclose(F, ref, atol=1e-13)
