"""Pins of the whole one-step scheme in the oracle (uniform grid, no GPU):
constant-state preservation, conservation, designed order on the isentropic
vortex, the exact Riemann solution of a shock tube, and the CFL
reading R1."""
import math

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W
from tests import exact_riemann as XR


def test_constant_state_preserved_bitwise_2d_3d():
    for d, M, n in [(2, 2, (6, 5)), (2, 3, (7, 8)), (3, 2, (5, 4, 6))]:
        o = O.Oracle(dim=d, degree=M, n=n, lo=(0,) * d, hi=(1,) * d, bc=(0,) * 6)
        o.set_initial(W.constant_state())
        u0 = o.get_cells()
        o.step(max_steps=2)
        assert np.array_equal(o.get_cells(), u0)


def test_dt_closed_form_rest_state():
    # R1: dt = CFL / max sum_dir (|v|+c)/dx ; rest state c = sqrt(1.4)
    o = O.Oracle(dim=2, degree=2, n=(8, 4), lo=(0, 0), hi=(2, 1), bc=(0,) * 6, cfl=0.9)
    o.set_initial(W.constant_state(rho=1.0, v=(0, 0, 0), p=1.0))
    c = math.sqrt(1.4)
    assert abs(o.compute_dt() - 0.9 / (c / 0.25 + c / 0.25)) < 1e-15


@pytest.mark.parametrize("d,M,n", [(2, 2, (12, 10)), (2, 3, (10, 9)), (3, 2, (6, 5, 4))])
def test_conservation_periodic(d, M, n):
    o = O.Oracle(dim=d, degree=M, n=n, lo=(0,) * d, hi=(1,) * d, bc=(0,) * 6, cfl=0.9)
    o.set_initial(W.random_smooth(d, seed=1212, amp=0.08))
    u0 = o.get_cells()
    o.step(max_steps=3)
    u1 = o.get_cells()
    tot0, tot1 = u0.sum(0), u1.sum(0)
    assert np.all(np.abs(tot1 - tot0) <= 1e-13 * u0.shape[0] * np.abs(u0).max(0))
    assert not np.array_equal(u0, u1)


def _vortex_err(n, M, t_end):
    o = O.Oracle(dim=2, degree=M, n=(n, n), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9)
    o.set_initial(W.isentropic_vortex())
    o.step(t_end, 10 ** 6)
    ex = O.Oracle(dim=2, degree=M, n=(n, n), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, ic_quad=M + 3)
    ex.set_initial(W.vortex_exact(t_end))
    e = o.get_cells()[:, 0] - ex.get_cells()[:, 0]
    h2 = (10.0 / n) ** 2
    return np.abs(e).sum() * h2, math.sqrt((e * e).sum() * h2)


@pytest.mark.parametrize("M,ns", [(2, (32, 64)), (3, (24, 48))])
def test_vortex_design_order(M, ns):
    # convergence of the isentropic vortex; design order M+1
    # (Table tab.conv2 reports 2.8-3.1 for O3 and 3.9-4.0 for O4).
    e1 = _vortex_err(ns[0], M, 0.25)
    e2 = _vortex_err(ns[1], M, 0.25)
    r = math.log(ns[1] / ns[0])
    o1, o2 = math.log(e1[0] / e2[0]) / r, math.log(e1[1] / e2[1]) / r
    assert o1 > M + 1 - 0.35 and o2 > M + 1 - 0.35, (o1, o2)


def test_sod_shock_tube_vs_exact_riemann():
    # 1D Riemann problem embedded in 2D (n x 1, periodic y, transmissive x),
    # compared with the exact solution; the L1 error must shrink with h.
    WL, WR = (1.0, 0.0, 1.0), (0.125, 0.0, 0.1)
    errs = []
    for n in (50, 100):
        o = O.Oracle(dim=2, degree=2, n=(n, 1), lo=(0, 0), hi=(1, 1.0 / n), bc=(1, 1, 0, 0, 0, 0), cfl=0.9)
        o.set_initial(W.shock_tube(0, 0.5))
        o.step(0.2, 10 ** 6)
        rho = o.get_cells()[:, 0]
        ref = XR.cell_average_density(WL, WR, 0.5, 0.2, np.linspace(0, 1, n + 1))
        errs.append(np.abs(rho - ref).mean())
    assert errs[0] < 0.02 and errs[1] < 0.6 * errs[0], errs


def test_transmissive_ghosts_keep_uniform_outflow():
    # uniform supersonic flow leaving through transmissive boundaries stays uniform
    o = O.Oracle(dim=2, degree=2, n=(8, 6), lo=(0, 0), hi=(1, 1), bc=(1,) * 6)
    o.set_initial(W.constant_state(rho=1.0, v=(2.0, 0.5, 0), p=0.5))
    u0 = o.get_cells()
    o.step(max_steps=2)
    np.testing.assert_allclose(o.get_cells(), u0, rtol=0, atol=1e-14)
