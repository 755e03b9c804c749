"""Pins of the oracle's Osher-type flux (eqn.osher @ P:186-196, Euler only).

The oracle builds |A| from the hand-differentiated Jacobian by Sylvester's
formula; nothing here re-types those formulas.  The Jacobian is pinned by
finite differences of the physical flux and by Euler homogeneity (A u = f);
|A| by numpy's general eigensolver (a different method) and by the
supersonic limits; the path integral by the fundamental theorem of calculus
(int_0^1 A(psi(s)) ds (uR - uL) = f(uR) - f(uL)), which the Gauss rule must
approach as nq grows; the scheme by the Sod tube against the exact Riemann
solution.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W
from tests import exact_riemann as XR

E = O.EULER


def _random_states(dim, n, seed=1212, vmax=1.0):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        pr = [rng.uniform(0.3, 2.0), *rng.uniform(-vmax, vmax, 3), rng.uniform(0.3, 2.0)]
        out.append(O.prim_to_cons(E, dim, 1.4, pr))
    return out


@pytest.mark.parametrize("dim", [2, 3])
def test_jacobian_matches_finite_differences(dim):
    for u in _random_states(dim, 6):
        for d in range(dim):
            A = O.euler_jacobian(dim, 1.4, u, d)
            J = np.zeros_like(A)
            for b in range(len(u)):
                h = 1e-6 * max(1.0, abs(u[b]))
                up, um = u.copy(), u.copy()
                up[b] += h
                um[b] -= h
                J[:, b] = (O.phys_flux(E, dim, 1.4, 0, up, d) - O.phys_flux(E, dim, 1.4, 0, um, d)) / (2 * h)
            np.testing.assert_allclose(A, J, rtol=1e-7, atol=1e-7)


@pytest.mark.parametrize("dim", [2, 3])
def test_jacobian_homogeneity(dim):
    # the Euler flux is homogeneous of degree one in u, so A(u) u = f(u)
    for u in _random_states(dim, 6, seed=3585):
        for d in range(dim):
            A = O.euler_jacobian(dim, 1.4, u, d)
            np.testing.assert_allclose(A @ u, O.phys_flux(E, dim, 1.4, 0, u, d), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_abs_jacobian_equals_eigendecomposition(dim):
    for u in _random_states(dim, 6):
        for d in range(dim):
            A = O.euler_jacobian(dim, 1.4, u, d)
            lam, R = np.linalg.eig(A)
            ref = (R * np.abs(lam.real)) @ np.linalg.inv(R)
            absA = O.euler_abs_jacobian(dim, 1.4, u, d)
            np.testing.assert_allclose(absA, ref.real, rtol=1e-9, atol=1e-10)
            # |A| commutes with A and squares to A^2
            np.testing.assert_allclose(absA @ A, A @ absA, atol=1e-11)
            np.testing.assert_allclose(absA @ absA, A @ A, atol=1e-10)


def test_abs_jacobian_supersonic_limits():
    c = math.sqrt(1.4)
    for sgn in (1, -1):
        u = O.prim_to_cons(E, 3, 1.4, [1.0, sgn * 2.5 * c, 0.3, -0.2, 1.0])
        A = O.euler_jacobian(3, 1.4, u, 0)
        np.testing.assert_allclose(O.euler_abs_jacobian(3, 1.4, u, 0), sgn * A, atol=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_osher_consistency(dim):
    for u in _random_states(dim, 5):
        for d in range(dim):
            np.testing.assert_array_equal(O.osher(dim, 1.4, u, u, d), O.phys_flux(E, dim, 1.4, 0, u, d))


def test_osher_supersonic_path_is_upwind():
    # all eigenvalues positive along the path: |A| = A, and the path integral
    # int A(psi(s)) ds (uR - uL) = f(uR) - f(uL), so the flux tends to f(uL)
    uL = O.prim_to_cons(E, 2, 1.4, [1.0, 3.0, 0.2, 0, 1.0])
    uR = O.prim_to_cons(E, 2, 1.4, [0.8, 3.2, -0.1, 0, 0.7])
    fL = O.phys_flux(E, 2, 1.4, 0, uL, 0)
    errs = [np.abs(O.osher(2, 1.4, uL, uR, 0, nq) - fL).max() for nq in (1, 2, 3, 6)]
    assert errs[-1] < 1e-12, errs
    assert errs[0] > errs[1] > errs[2], errs


def test_osher_small_jump_matches_linearisation():
    # int_0^1 |A(psi(s))| ds = |A(u_mid)| + O(|du|^2) away from sonic points
    u0 = O.prim_to_cons(E, 3, 1.4, [1.0, 0.3, -0.2, 0.1, 1.0])
    du = np.array([0.3, -0.2, 0.5, 0.1, 0.4])
    errs = []
    for eps in (1e-2, 5e-3):
        uL, uR = u0 - 0.5 * eps * du, u0 + 0.5 * eps * du
        lin = 0.5 * (O.phys_flux(E, 3, 1.4, 0, uL, 0) + O.phys_flux(E, 3, 1.4, 0, uR, 0)) \
            - 0.5 * O.euler_abs_jacobian(3, 1.4, u0, 0) @ (uR - uL)
        errs.append(np.abs(O.osher(3, 1.4, uL, uR, 0) - lin).max())
    assert errs[1] < errs[0] / 6, errs   # third order in eps


def test_osher_mirror_symmetry():
    pl = [1.0, 0.3, 0.1, 0, 1.0]
    prr = [0.5, -0.2, 0.4, 0, 0.4]
    uL, uR = O.prim_to_cons(E, 2, 1.4, pl), O.prim_to_cons(E, 2, 1.4, prr)
    mL = O.prim_to_cons(E, 2, 1.4, [prr[0], -prr[1], prr[2], 0, prr[4]])
    mR = O.prim_to_cons(E, 2, 1.4, [pl[0], -pl[1], pl[2], 0, pl[4]])
    F = O.osher(2, 1.4, uL, uR, 0)
    G = O.osher(2, 1.4, mL, mR, 0)
    np.testing.assert_allclose(G, [-F[0], F[1], -F[2], -F[3]], atol=1e-14)


def test_osher_rejected_for_mhd():
    with pytest.raises(ValueError):
        O.Oracle(dim=2, system=O.MHD, degree=2, n=(4, 4), lo=(0, 0), hi=(1, 1), bc=(0,) * 6, flux=O.OSHER)


def test_sod_tube_osher_vs_exact_riemann():
    # the scheme with the Osher flux converges to the exact Riemann solution and
    # is no more diffusive than the Rusanov scheme on the same grid
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    errs = {}
    for flux in (O.RUSANOV, O.OSHER):
        for n in (50, 100):
            o = O.Oracle(dim=2, degree=2, n=(n, 1), lo=(0, 0), hi=(1, 1.0 / n), bc=(1, 1, 0, 0, 0, 0), cfl=0.9,
                         flux=flux)
            o.set_initial(W.shock_tube(0, 0.5))
            o.step(0.2, 10 ** 6)
            ref = XR.cell_average_density(WL, WR, 0.5, 0.2, np.linspace(0, 1, n + 1))
            errs[flux, n] = np.abs(o.get_cells()[:, 0] - ref).mean()
    assert errs[O.OSHER, 50] < 0.02 and errs[O.OSHER, 100] < 0.6 * errs[O.OSHER, 50], errs
    assert errs[O.OSHER, 100] <= errs[O.RUSANOV, 100], errs


def test_osher_constant_state_and_conservation():
    o = O.Oracle(dim=2, degree=2, n=(8, 8), lo=(0, 0), hi=(1, 1), bc=(0,) * 6, flux=O.OSHER)
    o.set_initial(W.constant_state(rho=1.3, v=(0.4, -0.7, 0), p=0.9))
    u0 = o.get_cells()
    o.step(max_steps=2)
    np.testing.assert_array_equal(o.get_cells(), u0)
    o = O.Oracle(dim=2, degree=2, n=(8, 8), lo=(0, 0), hi=(1, 1), bc=(0,) * 6, flux=O.OSHER)
    o.set_initial(W.random_smooth(2, seed=3585, amp=0.2))
    u0 = o.get_cells()
    o.step(max_steps=3)
    u1 = o.get_cells()
    np.testing.assert_allclose(u1.sum(0), u0.sum(0), rtol=0, atol=1e-12 * np.abs(u0).sum(0).max())
    assert not np.array_equal(u0, u1)
