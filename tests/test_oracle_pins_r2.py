"""Round-2 pins of the oracle parts the round-1 review found unpinned (no GPU).

Each test checks the oracle against a value fixed by the mathematics, never
against a retyped copy of the oracle's own formula:

* AMR projection: child averages of random tensor polynomials of
  degree <= M in space and time against their closed-form integrals, every
  child position, several time fractions, 2D/3D, M = 2/3.
* Coarse-fine sub-face x sub-interval flux (eqn.memory.sum
  P:693-717): for a flux linear in the state (Euler entropy wave, v and p
  constant) the mapped space-time quadrature equals the exact average over
  the fine sub-face and sub-interval, and the flux memory summed over the
  r^(d-1) sub-faces and r sub-steps divided by r^d equals the coarse-face
  average.
* One AMR macro step on a linear entropy wave with two refinement levels is
  exact on every level (every stage of the scheme reproduces a linear
  solution: WENO and the predictor reproduce polynomials of degree <= M, the
  traces agree so the two-point flux is f(q), the Gauss rule is exact) — a
  swapped tangential axis, a wrong child offset, a wrong tau offset or a
  misplaced flux memory breaks it.
* MHD-GLM flux rows: the largest |eigenvalue| of the
  finite-difference Jacobian of the flux equals the oracle's max speed
  max(|v_n| + c_f, c_h) (the flux's GLM block is block-triangular, so its
  spectrum is the 7-wave MHD spectrum plus +-c_h), and a flux worked by hand
  at a state with v.B != 0 and Psi != 0.
* WENO constants r = 8 and eps = 1e-14: the oracle's one-dimensional
  reconstruction against an independent monomial-basis construction of the
  stencil polynomials, oscillation indicators integrated in closed form,
  on data where the indicators are O(1) (fixes r) and O(eps) (fixes eps);
  the test also shows that r = 6, 10 or eps = 1e-12, 1e-16 would fail.

tools/oracle_mutation_check.sh builds mutated copies of the oracle and shows
that these tests fail on each mutation (log: profiles/round2_oracle_mutations.log).
"""
import itertools
import math

import numpy as np
import pytest

import oracle as O

E, MHD = O.EULER, O.MHD


# ---------------------------------------------------------------------------
# helpers: nodal tensor polynomials on the Gauss-Legendre nodes
# ---------------------------------------------------------------------------

def _gl_nodes(N):
    # Gauss-Legendre nodes on [0,1] from numpy's Legendre module (independent
    # of the oracle's Newton iteration)
    x, _ = np.polynomial.legendre.leggauss(N)
    return 0.5 * (x + 1.0)


def _rand_poly(rng, nvar_axes, M):
    """coefficients c[a0, a1, ...] of sum c * prod x_k^a_k, degree <= M per axis"""
    return rng.normal(size=(M + 1,) * nvar_axes) * 0.3


def _eval_poly(c, xs):
    out = np.zeros_like(xs[0])
    for e in itertools.product(range(c.shape[0]), repeat=c.ndim):
        out = out + c[e] * np.prod([xs[k] ** e[k] for k in range(c.ndim)], axis=0)
    return out


def _mono_avg(a, lo, hi):
    # (1/(hi-lo)) int_lo^hi x^a dx
    return (hi ** (a + 1) - lo ** (a + 1)) / ((a + 1) * (hi - lo))


# ---------------------------------------------------------------------------
# AMR projection P:729-741
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("d,M,r", [(2, 2, 3), (2, 3, 3), (2, 3, 4), (3, 2, 3)])
def test_projection_into_every_child_is_the_exact_subbox_average(d, M, r):
    rng = np.random.default_rng(1212 + 10 * d + M)
    N = M + 1
    lam = _gl_nodes(N)
    idx = np.arange(N ** (d + 1))
    X = [lam[(idx // N ** k) % N] for k in range(d + 1)]     # x fastest, time slowest
    nv = 3
    C = [_rand_poly(rng, d + 1, M) for _ in range(nv)]
    q = np.array([_eval_poly(c, X) for c in C])                 # nodal = interpolant = the polynomial
    for off in itertools.product(range(r), repeat=d):
        for tau in [0.0, 1.0 / r, (r - 1.0) / r, 1.0, 0.37]:
            got = O.project_subbox(d, M, r, q, off[::-1] if False else off, tau, mode=1)
            ref = np.zeros(nv)
            for v in range(nv):
                for e in itertools.product(range(M + 1), repeat=d + 1):
                    term = C[v][e] * tau ** e[d]
                    for k in range(d):
                        term *= _mono_avg(e[k], off[k] / r, (off[k] + 1.0) / r)
                    ref[v] += term
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13 * max(1.0, np.abs(ref).max()),
                                       err_msg=f"child {off} tau {tau}")


@pytest.mark.parametrize("d,M", [(2, 2), (3, 2), (2, 3)])
def test_projection_of_the_weno_polynomial(d, M):
    # mode 0 (new active children take sub-box averages of w_h, reading R18)
    rng = np.random.default_rng(3585 + d + M)
    N, r = M + 1, 3
    lam = _gl_nodes(N)
    idx = np.arange(N ** d)
    X = [lam[(idx // N ** k) % N] for k in range(d)]
    c = _rand_poly(rng, d, M)
    w = _eval_poly(c, X)[None, :]
    tot = 0.0
    for off in itertools.product(range(r), repeat=d):
        got = O.project_subbox(d, M, r, w, off, 0.0, mode=0)[0]
        ref = 0.0
        for e in itertools.product(range(M + 1), repeat=d):
            term = c[e]
            for k in range(d):
                term *= _mono_avg(e[k], off[k] / r, (off[k] + 1.0) / r)
            ref += term
        assert abs(got - ref) <= 1e-13 * max(1.0, abs(ref)), (off, got, ref)
        tot += got
    # the r^d children average back to the mother's mean (eqn.average)
    mean = sum(c[e] * np.prod([1.0 / (e[k] + 1) for k in range(d)]) for e in itertools.product(range(M + 1), repeat=d))
    assert abs(tot / r ** d - mean) < 1e-13


# ---------------------------------------------------------------------------
# coarse-fine face: sub-face x sub-interval mapping and flux memory
# ---------------------------------------------------------------------------

def _entropy_cons(rho, v, p, g, d):
    nv = d + 2
    out = np.zeros((nv,) + np.shape(rho))
    out[0] = rho
    for k in range(d):
        out[1 + k] = rho * v[k]
    out[1 + d] = p / (g - 1) + 0.5 * rho * (v @ v)
    return out


def _euler_flux_of_rho(rbar, v, p, g, d, dirn):
    nv = d + 2
    f = np.zeros(nv)
    f[0] = rbar * v[dirn]
    for k in range(d):
        f[1 + k] = rbar * v[dirn] * v[k] + (p if k == dirn else 0.0)
    f[1 + d] = v[dirn] * (p / (g - 1) + 0.5 * rbar * (v @ v) + p)
    return f


@pytest.mark.parametrize("d,M,dirn,fine_side", [(2, 2, 0, 1), (2, 2, 1, 0), (2, 3, 0, 0), (3, 2, 2, 1), (3, 2, 1, 0)])
def test_coarse_fine_subface_flux_and_memory_sum(d, M, dirn, fine_side):
    """Coarse cell K = [0,1]^d over the time step [0,1]; fine cells of size 1/r
    on K's +dirn side (fine_side=1) or -dirn side (0), sub-step m in [m/r,(m+1)/r].
    rho(x, t) = 1 + a.x + at*t (physical = K's reference coordinates)."""
    r, g, p = 3, 1.4, 1.3
    N = M + 1
    lam = _gl_nodes(N)
    idx = np.arange(N ** (d + 1))
    X = [lam[(idx // N ** k) % N] for k in range(d + 1)]
    v = np.array([0.7, -0.4, 0.25])[:d]
    a = np.array([0.11, -0.07, 0.05])[:d]
    at = 0.03

    def rho(xs, t):
        return 1.0 + sum(a[k] * xs[k] for k in range(d)) + at * t
    qK = _entropy_cons(rho(X[:d], X[d]), v, p, g, d)
    tan = [k for k in range(d) if k != dirn]
    total = np.zeros(d + 2)
    for m in range(r):
        for c in itertools.product(range(r), repeat=d - 1):
            # fine cell F: reference xi -> physical x = x0 + xi / r, t = (m + tau) / r
            x0 = np.zeros(d)
            x0[dirn] = 1.0 if fine_side == 1 else -1.0 / r
            for j, k in enumerate(tan):
                x0[k] = c[j] / r
            qF = _entropy_cons(rho([x0[k] + X[k] / r for k in range(d)], (m + X[d]) / r), v, p, g, d)
            offK = np.zeros(3)
            for j, k in enumerate(tan):
                offK[k] = c[j] / r
            offK[dirn] = 1.0 if fine_side == 1 else 0.0
            offF = np.zeros(3)
            offF[dirn] = 0.0 if fine_side == 1 else 1.0
            if fine_side == 1:   # K is the lower (left) side of the face
                Ff = O.face_flux_mapped(d, M, E, g, 0, dirn, qK, offK, 1.0 / r, m / r, 1.0 / r,
                                        qF, offF, 1.0, 0.0, 1.0)
            else:
                Ff = O.face_flux_mapped(d, M, E, g, 0, dirn, qF, offF, 1.0, 0.0, 1.0,
                                        qK, offK, 1.0 / r, m / r, 1.0 / r)
            # exact average over the sub-face x sub-interval: rho is linear, the
            # flux linear in rho -> f(rho at the centre)
            xc = np.zeros(d)
            xc[dirn] = 1.0 if fine_side == 1 else 0.0
            for j, k in enumerate(tan):
                xc[k] = (c[j] + 0.5) / r
            ref = _euler_flux_of_rho(rho(xc, (m + 0.5) / r), v, p, g, d, dirn)
            np.testing.assert_allclose(Ff, ref, rtol=0, atol=2e-14, err_msg=f"m={m} c={c}")
            total += Ff
    # eqn.memory.sum: (1/r^d) sum of the fine fluxes = the coarse face average
    xc = np.full(d, 0.5)
    xc[dirn] = 1.0 if fine_side == 1 else 0.0
    coarse = _euler_flux_of_rho(rho(xc, 0.5), v, p, g, d, dirn)
    np.testing.assert_allclose(total / r ** d, coarse, rtol=0, atol=2e-14)
    # and the plain coarse-coarse face flux (full face, full step) agrees
    offL = np.zeros(3)
    offL[dirn] = 1.0 if fine_side == 1 else 0.0
    Fc = O.face_flux_mapped(d, M, E, g, 0, dirn, qK, offL, 1.0, 0.0, 1.0, None, np.zeros(3), 0, 0, 0) \
        if fine_side == 1 else O.face_flux_mapped(d, M, E, g, 0, dirn, None, np.zeros(3), 0, 0, 0, qK, offL, 1.0, 0.0, 1.0)
    np.testing.assert_allclose(Fc, coarse, rtol=0, atol=2e-14)


# ---------------------------------------------------------------------------
# one AMR macro step on a linear entropy wave is exact on every level
# ---------------------------------------------------------------------------

def _linear_wave(d, a, v, p):
    def ic(x):
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = 1.0 + x[:, :d] @ a
        out[:, 1:1 + d] = v
        out[:, 4] = p
        return out
    return ic


@pytest.mark.parametrize("d,M,lmax,n0,refine", [
    (2, 2, 2, 16, [(0, (7, 7)), (0, (8, 8)), (1, (23, 23))]),
    (2, 3, 2, 16, [(0, (7, 8)), (1, (22, 25))]),
    (3, 2, 1, 10, [(0, (4, 5, 4))]),
])
def test_amr_macro_step_exact_for_linear_entropy_wave(d, M, lmax, n0, refine):
    g, p = 1.4, 1.0
    a = np.array([0.2, -0.13, 0.07])[:d]
    v = np.array([0.5, -0.3, 0.2])[:d]
    A = O.AmrOracle(dim=d, degree=M, n=(n0,) * d, lo=(0,) * d, hi=(1,) * d, bc=(1,) * 6, lmax=lmax, cfl=0.45,
                    gamma=g)
    A.set_initial(_linear_wave(d, a, v, p))
    for lv, ix in refine:
        assert A.refine_cell(lv, ix) == 0
    lvl, st, ix, u0 = A.cells()
    assert (st[lvl == lmax] == 0).any(), "the finest level must hold active cells"
    rep = A.step(1e300, 1, adapt_every=0)
    t = rep.t
    lvl, st, ix, u = A.cells()
    r = 3
    dx0 = 1.0 / n0
    checked = np.zeros(lmax + 1, dtype=int)
    for i in np.where(st == 0)[0]:
        l = lvl[i]
        h = dx0 / r ** l
        anc = ix[i][:d] // r ** l
        if anc.min() < 4 or anc.max() > n0 - 5:   # transmissive boundary: ghosts are copies (R5)
            continue
        xc = (ix[i][:d] + 0.5) * h
        rho = 1.0 + (xc - v * t) @ a                 # linear: cell average = centre value
        ref = np.zeros(d + 2)
        ref[0] = rho
        ref[1:1 + d] = rho * v
        ref[1 + d] = p / (g - 1) + 0.5 * rho * (v @ v)
        assert np.abs(u[i] - ref).max() < 2e-14, (l, ix[i], u[i] - ref)
        checked[l] += 1
    assert (checked > 0).all(), checked


# ---------------------------------------------------------------------------
# MHD-GLM flux rows P:1427-1435
# ---------------------------------------------------------------------------

def test_mhd_jacobian_spectrum_matches_max_speed():
    rng = np.random.default_rng(1212)
    g = 5.0 / 3.0
    for trial in range(12):
        ch = [0.5, 2.0, 6.0][trial % 3]
        prim = [rng.uniform(0.5, 2.0), *rng.uniform(-1, 1, 3), rng.uniform(0.5, 2.0),
                *(rng.uniform(-1, 1, 3) * math.sqrt(4 * math.pi)), rng.uniform(-0.5, 0.5)]
        u = O.prim_to_cons(MHD, 2, g, prim)
        for dirn in (0, 1):
            J = np.zeros((9, 9))
            for j in range(9):
                h = 1e-6 * max(1.0, abs(u[j]))
                up, um = u.copy(), u.copy()
                up[j] += h
                um[j] -= h
                J[:, j] = (O.phys_flux(MHD, 2, g, ch, up, dirn) - O.phys_flux(MHD, 2, g, ch, um, dirn)) / (2 * h)
            ev = np.linalg.eigvals(J)
            assert np.abs(ev.imag).max() < 1e-5 * np.abs(ev).max(), ev    # hyperbolic: real spectrum
            smax = O.max_speed(MHD, 2, g, ch, u, dirn)
            assert abs(np.abs(ev.real).max() - smax) < 1e-6 * smax, (np.sort(ev.real), smax)
            # +-c_h are eigenvalues (GLM block)
            assert np.abs(ev.real - ch).min() < 1e-6 * ch and np.abs(ev.real + ch).min() < 1e-6 * ch


def test_mhd_flux_worked_by_hand():
    # state: rho = 2, v = (1, 1, 0), p = 1, B = sqrt(4 pi) (1, 0, 1), Psi = 0.5,
    # gamma = 5/3, c_h = 2.  With b = B / sqrt(4 pi) = (1, 0, 1):
    #   B^2/(8 pi) = |b|^2 / 2 = 1,  pt = p + 1 = 2,  v.B/(4 pi) -> b_n (v.b),
    #   E = p/(gamma-1) + rho |v|^2 / 2 + 1 = 1.5 + 2 + 1 = 4.5
    # x: (rho v_x, rho v_x^2 + pt - b_x^2, rho v_x v_y - b_x b_y, rho v_x v_z - b_x b_z,
    #     v_x (E + pt) - b_x (v.b), Psi, v_x B_y - B_x v_y, v_x B_z - B_x v_z, c_h^2 B_x)
    #   = (2, 2 + 2 - 1, 2, -1, 6.5 - 1, 0.5, -s, s, 4 s),  s = sqrt(4 pi)
    # y: (2, 2, 2 + 2, 0, 6.5 - 0, v_y B_x - B_y v_x, Psi, v_y B_z - B_y v_z, 0)
    #   = (2, 2, 4, 0, 6.5, s, 0.5, s, 0)
    s = math.sqrt(4 * math.pi)
    g, ch = 5.0 / 3.0, 2.0
    u = O.prim_to_cons(MHD, 2, g, [2, 1, 1, 0, 1, s, 0, s, 0.5])
    np.testing.assert_allclose(u, [2, 2, 2, 0, 4.5, s, 0, s, 0.5], rtol=0, atol=1e-14)
    np.testing.assert_allclose(O.phys_flux(MHD, 2, g, ch, u, 0), [2, 3, 2, -1, 5.5, 0.5, -s, s, 4 * s],
                               rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.phys_flux(MHD, 2, g, ch, u, 1), [2, 2, 4, 0, 6.5, s, 0.5, s, 0],
                               rtol=0, atol=1e-13)


# ---------------------------------------------------------------------------
# WENO constants r = 8, eps = 1e-14, lambda = 1e5 / 1
# ---------------------------------------------------------------------------

_STENCILS = {2: [(1, 1), (2, 0), (0, 2)], 3: [(2, 1), (1, 2), (3, 0), (0, 3)]}   # (L, R)


def _weno_reference(M, win, r=8, eps=1e-14, lam_c=1e5):
    """independent construction: monomial polynomial per stencil (its cell
    averages fixed), sigma = sum_alpha int_0^1 (p^(alpha))^2
     integrated exactly with numpy polynomials, weights of P:274."""
    N = M + 1
    nodes = _gl_nodes(N)
    base = win[M]                 # the reconstruction commutes with adding a constant
    win = np.asarray(win) - base  # (sigma ignores it): build it on the differences
    out = np.full(N, base)
    polys, sig, lin = [], [], []
    for (L, R) in _STENCILS[M]:
        offs = range(-L, R + 1)
        A = np.array([[_mono_avg(k, o, o + 1.0) for k in range(N)] for o in offs])
        c = np.linalg.solve(A, np.array([win[M + o] for o in offs]))
        P = np.polynomial.Polynomial(c)
        s = 0.0
        for al in range(1, M + 1):
            Q = (P.deriv(al) ** 2).integ()
            s += Q(1.0) - Q(0.0)
        polys.append(P)
        sig.append(s)
        lin.append(lam_c if L > 0 and R > 0 else 1.0)
    wt = np.array([lin[i] / (sig[i] + eps) ** r for i in range(len(sig))])
    wt /= wt.sum()
    for i, P in enumerate(polys):
        out += wt[i] * P(nodes)
    return out


@pytest.mark.parametrize("M", [2, 3])
def test_weno_weights_fix_r_and_eps(M):
    rng = np.random.default_rng(1212 + M)
    W = 2 * M + 1
    cases = []
    for _ in range(6):                       # O(1) indicators: the exponent r decides
        cases.append(1.0 + rng.uniform(-0.3, 0.3, W))
    for k in range(24, 33):                  # indicators ~ eps: eps decides (exact binary data)
        for _ in range(3):
            base = rng.integers(-8, 9, W).astype(float)
            cases.append(1.0 + base * 2.0 ** -k)
    for win in cases:
        got = O.weno_1d(M, win)
        ref = _weno_reference(M, win)
        spread = np.ptp(win)
        tol = 1e-12 * max(spread, 1e-10) + 2e-14
        assert np.abs(got - ref).max() <= tol, (win, got - ref)
    # discrimination: each other choice of the constants moves the result of
    # at least one case by more than 20x the tolerance
    for kw in (dict(r=6), dict(r=10), dict(eps=1e-12), dict(eps=1e-16), dict(lam_c=1e3)):
        assert any(np.abs(_weno_reference(M, w, **kw) - _weno_reference(M, w)).max()
                   > 20 * (1e-12 * max(np.ptp(w), 1e-10) + 2e-14) for w in cases), kw
