"""Pins of the time-dependent Dirichlet "exact solution prescribed" boundary
(reading R26: before every step the ghost layer
takes the cell averages of ic(x - t exact_vel)) and of the double Mach
reflection setup (reading R27) — no GPU."""
import math

import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W

EX = O.EXACT


def test_constant_state_with_exact_boundaries_is_bitwise_constant():
    o = O.Oracle(dim=2, degree=2, n=(12, 9), lo=(0, 0), hi=(1, 1), bc=(EX,) * 4, cfl=0.9,
                 exact_vel=(0.7, -0.3, 0))
    o.set_initial(W.constant_state())
    u0 = o.get_cells()
    o.step(1e300, 5)
    assert np.array_equal(o.get_cells(), np.tile(u0[0], (u0.shape[0], 1)))


def _traveling_wave_error(n, t_end, M):
    # smooth density wave advected by v at constant p: the exact solution is
    # the initial condition translated by v t, so exact_vel = v
    v = (0.8, 0.35, 0.0)
    ic = W.entropy_wave(2, amp=0.2, v=v, L=1.0)
    kw = dict(dim=2, degree=M, n=(n, n), lo=(0, 0), hi=(1, 1), bc=(EX,) * 4, cfl=0.9, exact_vel=v)
    o = O.Oracle(**kw)
    o.set_initial(ic)
    o.step(t_end, 10 ** 6)
    ex = O.Oracle(dim=2, degree=M, n=(n, n), lo=(-v[0] * t_end, -v[1] * t_end),
                  hi=(1 - v[0] * t_end, 1 - v[1] * t_end), bc=(0,) * 4, ic_quad=M + 3)
    ex.set_initial(ic)
    return np.abs(o.get_cells()[:, 0] - ex.get_cells()[:, 0]).mean()


@pytest.mark.parametrize("M,min_order", [(2, 2.6), (3, 3.5)])
def test_traveling_wave_through_exact_boundaries_converges_at_design_order(M, min_order):
    # the wave leaves through two sides and enters through the other two; with
    # the ghost layers from the exact solution the scheme keeps its order M+1
    e1 = _traveling_wave_error(12, 0.25, M)
    e2 = _traveling_wave_error(24, 0.25, M)
    order = math.log(e1 / e2) / math.log(2.0)
    assert order > min_order, (e1, e2, order)


def test_dmr_initial_condition_and_front():
    # reading R27: the front line x = 1/6 + y / sqrt(3), post-shock state behind it,
    # and the exact solution translated with the Mach-10 front velocity
    ic = W.double_mach_reflection()
    ys = np.linspace(0, 1, 11)
    xs = 1 / 6 + ys / math.sqrt(3)
    before = ic(np.stack([xs - 1e-9, ys, 0 * ys], 1))
    after = ic(np.stack([xs + 1e-9, ys, 0 * ys], 1))
    assert np.all(before[:, 0] == 8.0) and np.all(after[:, 0] == 1.4)
    vel = np.array(W.DMR_FRONT_VEL[:2])
    assert abs(np.linalg.norm(vel) - 10.0) < 1e-14
    # the post-shock velocity is along the front normal (towards the pre-shock gas)
    assert abs(before[0, 1] * vel[1] - before[0, 2] * vel[0]) < 1e-12 and before[0, 1] * vel[0] > 0
    # Rankine-Hugoniot: mass flux through the moving front is continuous
    un = lambda s: (s[1] * vel[0] + s[2] * vel[1]) / 10.0
    m_post = before[0, 0] * (un(before[0]) - 10.0)
    m_pre = after[0, 0] * (un(after[0]) - 10.0)
    assert abs(m_post - m_pre) / abs(m_pre) < 2e-3   # 8.25 and 116.5 are the paper's rounded values


def test_dmr_mach10_is_inadmissible_with_the_literal_bottom_wall():
    # reading R27: the paper's bottom "reflective wall" meets the
    # post-shock inflow left of the shock foot; the unlimited reconstruction of
    # the Mach-10 jump there is inadmissible in the first step
    wl = W.config("dmr", 60)
    o = O.Oracle(dim=2, degree=2, n=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=wl.cfl,
                 exact_vel=wl.extra["exact_vel"])
    o.set_initial(wl.ic)
    with pytest.raises(RuntimeError, match="cell \\([34],0,0\\)"):
        o.step(wl.t_end, 10 ** 6)


def test_dmr_states_reproduce_the_paper_at_mach_10():
    post, pre, speed = W.dmr_states(10.0)
    assert abs(post[0] - 8.0) < 1e-12 and abs(post[2] - 116.5) < 1e-12 and abs(post[1] - 8.25) < 1e-12
    assert pre == (1.4, 0.0, 1.0) and speed == 10.0


def test_dmr_top_boundary_tracks_the_moving_shock():
    # the top row follows the exact solution: far from the reflection, the
    # shock (Mach M) crosses y = 1 at x_s(t) = 1/6 + (1 + 2 M t) / sqrt(3)
    wl = W.config("dmr2", 60)
    mach = wl.extra["mach"]
    o = O.Oracle(dim=2, degree=2, n=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=wl.cfl,
                 exact_vel=wl.extra["exact_vel"])
    o.set_initial(wl.ic)
    o.step(0.5, 10 ** 6)
    t = o.t
    post, pre, _ = W.dmr_states(mach)
    u = o.get_cells().reshape(wl.n[1], wl.n[0], 4)
    top = u[-1, :, 0]
    dx = 3.0 / wl.n[0]
    xc = (np.arange(wl.n[0]) + 0.5) * dx
    xs = 1 / 6 + (1 + 2 * mach * t) / math.sqrt(3)
    front = xc[np.argmax(top < 0.5 * (post[0] + pre[0]))]
    assert abs(front - xs) < 2 * dx, (front, xs)
    assert np.all(np.abs(top[xc < xs - 3 * dx] - post[0]) < 0.05 * post[0])
    assert np.all(np.abs(top[xc > xs + 3 * dx] - pre[0]) < 1e-4 * pre[0])
    assert np.all(np.abs(top[xc > xs + 12 * dx] - pre[0]) < 1e-13)   # undisturbed gas ahead
