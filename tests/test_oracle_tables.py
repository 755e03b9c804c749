"""Pins of the oracle's basis tables, WENO and predictor operators against
closed forms and brute force (no GPU).  Each test names the paper passage
whose definition it pins (P:n = PAPER.md line n)."""
import math

import numpy as np
import pytest

import oracle as O


def test_gauss_legendre_closed_forms():
    # nodes of the nodal basis are the M+1 Gauss-Legendre nodes on [0,1]
    t = O.tables(2)
    s = math.sqrt(15.0) / 10.0
    np.testing.assert_allclose(t["lam"], [0.5 - s, 0.5, 0.5 + s], rtol=0, atol=2e-16)
    np.testing.assert_allclose(t["w"], [5 / 18, 4 / 9, 5 / 18], rtol=0, atol=2e-16)
    t = O.tables(3)
    a = math.sqrt(3 / 7 - 2 / 7 * math.sqrt(6 / 5))
    b = math.sqrt(3 / 7 + 2 / 7 * math.sqrt(6 / 5))
    np.testing.assert_allclose(t["lam"], [0.5 - b / 2, 0.5 - a / 2, 0.5 + a / 2, 0.5 + b / 2], atol=3e-16)
    wa, wb = (18 + math.sqrt(30)) / 72, (18 - math.sqrt(30)) / 72
    np.testing.assert_allclose(t["w"], [wb, wa, wa, wb], atol=3e-16)


@pytest.mark.parametrize("M", [2, 3])
def test_mass_is_diagonal_and_lagrange_property(M):
    # psi_l(lambda_k) = delta_lk -> orthogonal basis, diagonal GL mass
    t = O.tables(M)
    np.testing.assert_allclose(t["M1"], np.diag(t["w"]), atol=1e-15)


def test_derivative_matrix_closed_form_M2():
    # K^xi 1D factor int psi_a psi_b' = w_a psi_b'(lambda_a) (GL exactness);
    # closed form D = sqrt(15)/3 [[-3,4,-1],[-1,0,1],[1,-4,3]]
    t = O.tables(2)
    D = t["Kx1"] / t["w"][:, None]
    Dref = math.sqrt(15.0) / 3.0 * np.array([[-3, 4, -1], [-1, 0, 1], [1, -4, 3]], dtype=float)
    np.testing.assert_allclose(D, Dref, atol=2e-14)


@pytest.mark.parametrize("M", [2, 3])
def test_time_operator_properties(M):
    # K1 time block.  A constant-in-time q with zero flux solves the
    # weak problem with initial data w: K1t^-1 psi(0) = 1.
    t = O.tables(M)
    K1t = t["K1t"]
    np.testing.assert_allclose(np.linalg.solve(K1t, t["psi0"]), np.ones(M + 1), atol=1e-13)
    # T = K1t^-1 diag(w) integrates in time: (T g)(lambda_s) = int_0^lambda_s g
    # exactly for polynomials g of degree <= M-1 (DG in time with upwind trace).
    T = np.linalg.solve(K1t, np.diag(t["w"]))
    lam = t["lam"]
    for k in range(M):
        np.testing.assert_allclose(T @ ((k + 1) * lam ** k), lam ** (k + 1), atol=1e-13)
    # App. A.5 of SURVEY prints T for M=2
    if M == 2:
        Tref = np.array([[0.16111111, -0.080421112, 0.032011666],
                         [0.27248542, 0.27777778, -0.050263195],
                         [0.29021056, 0.43597667, 0.16111111]])
        np.testing.assert_allclose(T, Tref, atol=1e-8)


@pytest.mark.parametrize("M", [2, 3])
def test_sigma_on_monomials(M):
    # eqn.sigmas / Sigma_pm = sum_alpha int psi_p^(a) psi_m^(a):
    # for nodal coefficients of p(xi) it returns sum_alpha int (p^(alpha))^2.
    t = O.tables(M)
    lam = t["lam"]
    S = t["Sigma"]
    for coeffs, ref in [((1.0,), 0.0), ((0.0, 1.0), 1.0), ((0.0, 0.0, 1.0), 4 / 3 + 4.0)]:
        c = np.polynomial.polynomial.polyval(lam, coeffs)
        assert abs(c @ S @ c - ref) < 1e-11 * max(1.0, ref)
    if M == 3:
        c = lam ** 3
        assert abs(c @ S @ c - (9 / 5 + 12 + 36)) < 1e-10


def test_jiang_shu_smoothness_indicators_M2():
    # For M=2 the indicators reduce to the Jiang-Shu forms:
    # central:  1/4 (c-a)^2 + 13/12 (a-2b+c)^2 ; left-sided on (a,b,c) = (u_{i-2},u_{i-1},u_i):
    # 1/4 (a-4b+3c)^2 + 13/12 (a-2b+c)^2 ; right-sided on (u_i,u_{i+1},u_{i+2}):
    # 1/4 (3a-4b+c)^2 + 13/12 (a-2b+c)^2
    t = O.tables(2)
    rng = np.random.default_rng(1212)
    for _ in range(20):
        a, b, c = rng.normal(size=3)
        for s, ref in [(0, 0.25 * (c - a) ** 2 + 13 / 12 * (a - 2 * b + c) ** 2),
                       (1, 0.25 * (a - 4 * b + 3 * c) ** 2 + 13 / 12 * (a - 2 * b + c) ** 2),
                       (2, 0.25 * (3 * a - 4 * b + c) ** 2 + 13 / 12 * (a - 2 * b + c) ** 2)]:
            w = t["rec"][s] @ np.array([a, b, c])
            assert abs(w @ t["Sigma"] @ w - ref) < 1e-11 * (1 + abs(ref))


def test_central_nodal_values_M2():
    # closed form of the central M=2 stencil polynomial at the GL nodes
    t = O.tables(2)
    rng = np.random.default_rng(3585)
    for _ in range(10):
        a, b, c = rng.normal(size=3)
        w = t["rec"][0] @ np.array([a, b, c])
        k = math.sqrt(15) / 20
        ref = [b - k * (c - a) + (a - 2 * b + c) / 30, b - (a - 2 * b + c) / 24, b + k * (c - a) + (a - 2 * b + c) / 30]
        np.testing.assert_allclose(w, ref, atol=1e-13)


@pytest.mark.parametrize("M", [2, 3])
def test_stencil_inverse_brute_force(M):
    # eqn.rec.x solved independently in the monomial basis:
    # find c_j with (1/1) int_o^{o+1} sum_j c_j xi^j = u_o for the stencil cells,
    # evaluate at the nodes, compare with Rec_s u.
    t = O.tables(M)
    rng = np.random.default_rng(1212)
    for s in range(t["nS"]):
        L, R = int(t["L"][s]), int(t["R"][s])
        offs = np.arange(-L, R + 1)
        A = np.array([[((o + 1.0) ** (j + 1) - o ** (j + 1.0)) / (j + 1) for j in range(M + 1)] for o in offs])
        u = rng.normal(size=M + 1)
        coef = np.linalg.solve(A, u)
        ref = np.polynomial.polynomial.polyval(t["lam"], coef)
        np.testing.assert_allclose(t["rec"][s] @ u, ref, atol=1e-11)
    # stencil shapes, eqn.stencildef @ P:220-224
    if M == 2:
        assert [(int(a), int(b)) for a, b in zip(t["L"], t["R"])] == [(1, 1), (2, 0), (0, 2)]
        assert list(t["lin"]) == [1e5, 1.0, 1.0]
    else:
        assert [(int(a), int(b)) for a, b in zip(t["L"], t["R"])] == [(2, 1), (1, 2), (3, 0), (0, 3)]
        assert list(t["lin"]) == [1e5, 1e5, 1.0, 1.0]


def _poly_cell_avgs(coef, centers_lo):
    # exact averages of a 1D polynomial on unit cells [o, o+1]
    P = np.polynomial.polynomial.polyint(coef)
    return np.array([np.polynomial.polynomial.polyval(o + 1.0, P) - np.polynomial.polynomial.polyval(o, P) for o in centers_lo])


@pytest.mark.parametrize("M", [2, 3])
def test_weno_1d_exact_on_polynomials_and_conservative(M):
    t = O.tables(M)
    rng = np.random.default_rng(3585)
    for _ in range(5):
        coef = rng.normal(size=M + 1)
        win = _poly_cell_avgs(coef, np.arange(-M, M + 1))
        out = O.weno_1d(M, win)
        np.testing.assert_allclose(out, np.polynomial.polynomial.polyval(t["lam"], coef), atol=1e-11)
    for _ in range(20):   # arbitrary (even discontinuous) data keeps the cell mean
        win = rng.normal(size=2 * M + 1) * rng.choice([1.0, 100.0], size=2 * M + 1)
        out = O.weno_1d(M, win)
        assert abs(t["w"] @ out - win[M]) < 1e-12 * (1 + np.abs(win).max())


def test_weno_non_oscillatory_at_jump():
    # near a discontinuity the smooth one-sided stencil dominates: for data
    # (1,1,1,0,0) centred on the last cell of the plateau the left stencil is exact
    out = O.weno_1d(2, np.array([1.0, 1.0, 1.0, 0.0, 0.0]))
    assert np.all(out <= 1.0 + 1e-6) and np.all(out >= 1.0 - 1e-3)


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_box_reconstruction_exact_for_tensor_polynomials(d, M):
    # dimension-by-dimension reconstruction is exact for
    # polynomials of degree <= M in each variable
    t = O.tables(M)
    rng = np.random.default_rng(1212)
    W = 2 * M + 1
    cs = [rng.normal(size=M + 1) for _ in range(d)]
    av = [_poly_cell_avgs(c, np.arange(-M, M + 1)) for c in cs]
    nv = 2
    if d == 2:
        box = np.einsum("j,i->ji", av[1], av[0]).reshape(-1)
    else:
        box = np.einsum("k,j,i->kji", av[2], av[1], av[0]).reshape(-1)
    ub = np.stack([box, 2 * box + 1], axis=1)
    w = O.reconstruct_box(d, M, nv, ub)
    vals = [np.polynomial.polynomial.polyval(t["lam"], c) for c in cs]
    ref = np.einsum("j,i->ji", vals[1], vals[0]).reshape(-1) if d == 2 else \
        np.einsum("k,j,i->kji", vals[2], vals[1], vals[0]).reshape(-1)
    np.testing.assert_allclose(w[0], ref, atol=1e-10)
    np.testing.assert_allclose(w[1], 2 * ref + 1, atol=1e-10)


@pytest.mark.parametrize("d,M", [(2, 2), (3, 2), (2, 3)])
def test_dense_predictor_operators_structure(d, M):
    # K1 is block diagonal in space with time blocks w_x K1t
    # (P:472-474), F0 maps a spatial field to psi_s(0) w_x values.
    t = O.tables(M)
    K1, Kd, F0 = O.predictor_matrices(d, M)
    N = M + 1
    NS = N ** d
    lam = t["lam"]
    # K^xi applied to a field linear in xi returns w_node * 1 (exact derivative)
    # coordinate arrays in x-fastest order
    idx = np.arange(NS * N)
    coords = [(idx // N ** k) % N for k in range(d + 1)]
    wnode = np.prod([t["w"][c] for c in coords], axis=0)
    for dirn in range(d):
        f = lam[coords[dirn]]
        np.testing.assert_allclose(Kd[dirn] @ f, wnode, atol=1e-13)
    # K1^-1 F0 w = w at every time node (the constant-in-time solution)
    wsp = np.random.default_rng(1).normal(size=NS)
    q = np.linalg.solve(K1, F0 @ wsp)
    np.testing.assert_allclose(q, np.tile(wsp, N), atol=1e-12)


@pytest.mark.parametrize("M", [2, 3])
def test_weno_linear_weights_on_near_constant_data(M):
    # R13: in smooth regions with sigma << eps = 1e-14 the nonlinear
    # weights reduce to the linear ones; the oscillation indicator must not be
    # swamped by round-off of the O(1) dofs (data 3.5 + 1e-9 sin).
    t = O.tables(M)
    x = np.arange(-M, M + 1)
    win = 3.5 + 1e-9 * np.sin(0.7 * x + 0.3)
    out = O.weno_1d(M, win)
    lin = t["lin"] / t["lin"].sum()
    ref = sum(lin[s] * (t["rec"][s] @ win[M - t["L"][s]: M + t["R"][s] + 1]) for s in range(t["nS"]))
    np.testing.assert_allclose(out, ref, rtol=0, atol=2e-15)
