"""Pins of the predictor initial guess (reading R25:
the previous step's q_h of the cell extrapolated in time, anchored at the new
reconstruction) — no GPU."""
import itertools

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W

E = O.EULER


def _gl(N):
    x, _ = np.polynomial.legendre.leggauss(N)
    return 0.5 * (x + 1.0)


@pytest.mark.parametrize("d,M,r", [(2, 2, 1.0), (2, 3, 0.7), (3, 2, 1.3)])
def test_extrapolation_is_exact_for_polynomials_in_time(d, M, r):
    # P(x, t) of degree <= M per variable; old step [t0, t0 + h1], new step
    # [t0 + h1, t0 + h1 + h2] with h2 = r h1: the guess at the new nodes is
    # P itself (evaluated directly, not through the Lagrange basis)
    rng = np.random.default_rng(1212 + d + M)
    N = M + 1
    lam = _gl(N)
    idx = np.arange(N ** (d + 1))
    X = [lam[(idx // N ** k) % N] for k in range(d + 1)]
    nv = 2
    C = rng.normal(size=(nv,) + (M + 1,) * (d + 1)) * 0.3
    t0, h1 = 0.37, 0.8
    h2 = r * h1

    def P(v, xs, t):
        out = np.zeros_like(t)
        for e in itertools.product(range(M + 1), repeat=d + 1):
            out = out + C[v][e] * np.prod([xs[k] ** e[k] for k in range(d)], axis=0) * t ** e[d]
        return out
    xs = X[:d]
    qp = np.array([P(v, xs, t0 + h1 * X[d]) for v in range(nv)])
    ns = N ** d
    w = np.array([P(v, [x[:ns] for x in xs], np.full(ns, t0 + h1)) for v in range(nv)])
    q0 = O.extrapolate_guess(d, M, w, qp, r)
    ref = np.array([P(v, xs, t0 + h1 + h2 * X[d]) for v in range(nv)])
    np.testing.assert_allclose(q0, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_exact_guess_converges_in_one_sweep(d, M):
    # entropy wave (flux linear in rho): the exact space-time polynomial is the
    # fixed point, so started from it the Picard iteration stops after one
    # sweep at the same result as from the time-constant guess (R3)
    N = M + 1
    lam = _gl(N)
    idx = np.arange(N ** (d + 1))
    X = [lam[(idx // N ** k) % N] for k in range(d + 1)]
    v = np.array([0.7, -0.4, 0.25])[:d]
    a = np.array([0.11, -0.07, 0.05])[:d]
    p, g = 1.3, 1.4
    dtdx = np.array([0.35, 0.3, 0.25])[:d]
    nv = d + 2

    def cons(rho):
        out = np.zeros((nv, rho.size))
        out[0] = rho
        for k in range(d):
            out[1 + k] = rho * v[k]
        out[1 + d] = p / (g - 1) + 0.5 * rho * (v @ v)
        return out
    ns = N ** d
    w = cons(1.0 + sum(a[k] * X[k][:ns] for k in range(d)))
    exact = cons(1.0 + sum(a[k] * (X[k] - v[k] * dtdx[k] * X[d]) for k in range(d)))
    rc0, q_r3, sw_r3 = O.predict_cell(d, M, E, g, 0, w, dtdx)
    rc1, q_g, sw_g = O.predict_cell(d, M, E, g, 0, w, dtdx, q0=exact)
    assert rc0 == 0 and rc1 == 0
    assert sw_g == 1 and sw_r3 > 1
    np.testing.assert_allclose(q_g, q_r3, rtol=0, atol=1e-12)


def test_guess_run_matches_and_saves_sweeps():
    # the vortex at order 4: the same solution within the Picard tolerance's
    # reach, fewer sweeps
    # (the first step has no previous step; on 32^2 the next 3 steps take
    # 8.14 sweeps per cell from R3, 7.92 from R25)
    kw = dict(dim=2, degree=3, n=(32, 32), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9)
    a = O.Oracle(**kw)
    b = O.Oracle(pred_guess=1, **kw)
    a.set_initial(W.isentropic_vortex())
    b.set_initial(W.isentropic_vortex())
    a.step(1e300, 1)
    b.step(1e300, 1)
    ra = a.step(1e300, 3)
    rb = b.step(1e300, 3)
    ua, ub = a.get_cells(), b.get_cells()
    assert (np.abs(ua - ub).max(axis=0) / np.abs(ua).max(axis=0)).max() < 1e-11
    assert rb.sweeps_total < ra.sweeps_total, (rb.sweeps_total, ra.sweeps_total)
