"""Pins of the oracle's Dirichlet inflow boundary (reading R23, SURVEY §8f #3:
the inflow sides of the double Mach reflection / forward step).

An inflow side keeps the ghost layer at the initial condition's cell averages
(the IC callback evaluated beyond the boundary), so a Riemann problem whose
discontinuity sits on the boundary must converge to the exact Riemann solution
restricted to the domain, and a state that equals its inflow is preserved.
"""
import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W
from tests import exact_riemann as XR

T, P, I = O.TRANSMISSIVE, O.PERIODIC, O.INFLOW


def test_inflow_of_the_same_state_is_steady():
    o = O.Oracle(dim=2, degree=2, n=(9, 6), lo=(0, 0), hi=(1, 1), bc=(I, T, P, P, 0, 0), cfl=0.9)
    o.set_initial(W.constant_state(rho=1.2, v=(0.7, 0.1, 0.0), p=0.9))
    u0 = o.get_cells()
    o.step(1e300, 4)
    np.testing.assert_allclose(o.get_cells(), u0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("M", [2, 3])
def test_riemann_problem_on_the_inflow_boundary(M):
    # left state held in the inflow ghosts, right state in the domain: the
    # solution is the exact Riemann fan restricted to x > 0
    WL, WR = (1.0, 0.75, 1.0), (0.125, 0.0, 0.1)
    errs = []
    for n in (40, 80):
        o = O.Oracle(dim=2, degree=M, n=(n, 1), lo=(0, 0), hi=(1, 1.0 / n), bc=(I, T, P, P, 0, 0), cfl=0.5)
        o.set_initial(W.shock_tube(0, 0.0, left=WL, right=WR))
        o.step(0.2, 10 ** 6)
        ref = XR.cell_average_density(WL, WR, 0.0, 0.2, np.linspace(0, 1, n + 1))
        errs.append(np.abs(o.get_cells()[:, 0] - ref).mean())
    assert errs[0] < 0.03 and errs[1] < 0.7 * errs[0], errs


def test_inflow_rejected_for_amr():
    with pytest.raises(ValueError):
        O.AmrOracle(dim=2, degree=2, n=(8, 8), lo=(0, 0), hi=(1, 1), bc=(I, T, P, P, 0, 0), lmax=1)
