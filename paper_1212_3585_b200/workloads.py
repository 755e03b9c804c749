"""Seeded, synthetic inputs shared by the CUDA path and the oracle.

This module holds ONLY input specifications: the paper's initial conditions as
point functions x -> primitive state, and the workload configurations of
BASELINE.json.  It holds none of the method's arithmetic (no reconstruction,
predictor, flux, update, quadrature or basis table); both the CUDA library and
the oracle call these point functions through their own IC callbacks and do
their own cell averaging.

Primitive layout of every IC: (rho, vx, vy, vz, p, Bx, By, Bz, psi).

Citations: P:n = PAPER.md line n.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEEDS = (1212, 3585)


# --------------------------------------------------------------------------
# Initial conditions
# --------------------------------------------------------------------------

def isentropic_vortex(eps=5.0, gamma=1.4, center=(5.0, 5.0)):
    """2D isentropic vortex, eq:pert @ P:875-896 (eps = 5, gamma = 1.4)."""
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        dx = x[:, 0] - center[0]
        dy = x[:, 1] - center[1]
        r2 = dx * dx + dy * dy
        dT = -(eps * eps * (gamma - 1.0)) / (8.0 * gamma * math.pi ** 2) * np.exp(1.0 - r2)
        e = eps / (2.0 * math.pi) * np.exp(0.5 * (1.0 - r2))
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = (1.0 + dT) ** (1.0 / (gamma - 1.0))
        out[:, 1] = 1.0 - dy * e
        out[:, 2] = 1.0 + dx * e
        out[:, 4] = (1.0 + dT) ** (gamma / (gamma - 1.0))
        return out
    return ic


def vortex_exact(t, eps=5.0, gamma=1.4, period=10.0):
    """Exact solution of the vortex at time t: advection by (1,1) on the periodic [0,10]^2."""
    base = isentropic_vortex(eps, gamma)

    def ic(x):
        y = np.array(x, dtype=np.float64, copy=True)
        y[:, 0] = np.mod(y[:, 0] - t, period)
        y[:, 1] = np.mod(y[:, 1] - t, period)
        return base(y)
    return ic


def explosion(dim, radius=0.5, inner=(1.0, 1.0), outer=(0.125, 0.1)):
    """Cylindrical/spherical explosion, P:995-1024 and Table tab.3d.explos.ic
    (rho, p) = (1, 1) inside r <= R, (0.125, 0.1) outside, zero velocity.
    BASELINE.json uses R = 0.5 (the paper's R = 0.4 is reading D2)."""
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        r2 = np.zeros(x.shape[0])
        for k in range(dim):
            r2 += x[:, k] * x[:, k]
        inside = r2 <= radius * radius
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = np.where(inside, inner[0], outer[0])
        out[:, 4] = np.where(inside, inner[1], outer[1])
        return out
    return ic


def orszag_tang(gamma=5.0 / 3.0):
    """Orszag-Tang vortex, B scaled by sqrt(4 pi) (Gaussian units)."""
    s = math.sqrt(4.0 * math.pi)

    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = gamma * gamma
        out[:, 1] = -np.sin(x[:, 1])
        out[:, 2] = np.sin(x[:, 0])
        out[:, 4] = gamma
        out[:, 5] = -s * np.sin(x[:, 1])
        out[:, 6] = s * np.sin(2.0 * x[:, 0])
        return out
    return ic


def shock_tube(axis=0, x0=0.5, left=(1.0, 0.0, 1.0), right=(0.125, 0.0, 0.1)):
    """Sod-type Riemann problem along one axis (rho, v_n, p) (test-only workload)."""
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        lft = x[:, axis] < x0
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = np.where(lft, left[0], right[0])
        out[:, 1 + axis] = np.where(lft, left[1], right[1])
        out[:, 4] = np.where(lft, left[2], right[2])
        return out
    return ic


# Double Mach reflection (eqn.dmr.ic), reading R27: the shock
# front is the line x' = (x - 1/6) cos(a) - y sin(a) = 0 with a = 30 degrees
# (the line through (1/6, 0) at 60 degrees to the x axis, the paper's
# "inclination angle of 60 degrees"), post-shock for x' < 0 with velocity
# 8.25 (cos a, -sin a) along the front normal (the paper prints +8.25 sin a,
# which would point the post-shock flow away from the shock it comes from),
# pre-shock (1.4, 0, 0, 0, 1).  The front moves with the Mach-10 shock speed
# 10 (pre-shock sound speed 1) along its normal: DMR_FRONT_VEL = 10 (cos a, -sin a).
DMR_ALPHA = math.pi / 6.0
DMR_FRONT_VEL = (10.0 * math.cos(DMR_ALPHA), -10.0 * math.sin(DMR_ALPHA), 0.0)


def dmr_states(mach=10.0, gamma=1.4):
    """(post (rho, u_n, p), pre (rho, 0, p), front speed) of a shock of Mach
    number `mach` into (rho, p) = (1.4, 1) (sound speed 1), Rankine-Hugoniot.
    mach = 10 gives the paper's printed (8, 8.25, 116.5)."""
    r1, p1 = 1.4, 1.0
    m2 = mach * mach
    r2 = r1 * (gamma + 1.0) * m2 / ((gamma - 1.0) * m2 + 2.0)
    p2 = p1 * (1.0 + 2.0 * gamma / (gamma + 1.0) * (m2 - 1.0))
    u2 = mach * (1.0 - r1 / r2)
    return (r2, u2, p2), (r1, 0.0, p1), mach


def double_mach_reflection(mach=10.0):
    """the paper's states at mach = 10 (printed values); other
    Mach numbers from dmr_states (the same geometry)"""
    ca, sa = math.cos(DMR_ALPHA), math.sin(DMR_ALPHA)
    if mach == 10.0:
        post, pre = (8.0, 8.25, 116.5), (1.4, 0.0, 1.0)
    else:
        post, pre, _ = dmr_states(mach)

    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        xp = (x[:, 0] - 1.0 / 6.0) * ca - x[:, 1] * sa
        ps = xp < 0.0
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = np.where(ps, post[0], pre[0])
        out[:, 1] = np.where(ps, post[1] * ca, 0.0)
        out[:, 2] = np.where(ps, -post[1] * sa, 0.0)
        out[:, 4] = np.where(ps, post[2], pre[2])
        return out
    return ic


def dmr_front_vel(mach=10.0):
    return (mach * math.cos(DMR_ALPHA), -mach * math.sin(DMR_ALPHA), 0.0)


def constant_state(rho=1.0, v=(0.3, -0.2, 0.1), p=0.7, B=(0.0, 0.0, 0.0)):
    def ic(x):
        out = np.zeros((np.asarray(x).shape[0], 9))
        out[:, 0] = rho
        out[:, 1:4] = v
        out[:, 4] = p
        out[:, 5:8] = B
        return out
    return ic


def entropy_wave(dim, amp=0.2, v=(1.0, 0.5, 0.25), p=1.0, L=1.0):
    """Density wave advected by a constant velocity at constant pressure."""
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        ph = np.zeros(x.shape[0])
        for k in range(dim):
            ph += 2.0 * math.pi * x[:, k] / L
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = 1.0 + amp * np.sin(ph)
        out[:, 1:1 + dim] = v[:dim]
        out[:, 4] = p
        return out
    return ic


def random_smooth(dim, seed=SEEDS[0], modes=3, amp=0.05, system=0):
    """Seeded smooth random admissible state (sum of a few Fourier modes)."""
    rng = np.random.default_rng(seed)
    coef = rng.uniform(-1.0, 1.0, size=(9, modes, dim))
    phase = rng.uniform(0.0, 2 * math.pi, size=(9, modes))
    base = np.array([1.0, 0.2, -0.1, 0.05, 1.0, 0.3, 0.2, -0.1, 0.0])

    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        out = np.tile(base, (x.shape[0], 1))
        for v in range(9):
            for m in range(modes):
                arg = phase[v, m] + 2.0 * math.pi * (x[:, :dim] @ np.round(coef[v, m] * 2.0))
                out[:, v] += amp * np.sin(arg)
        if system == 0:
            out[:, 5:] = 0.0
        if dim == 2:
            out[:, 3] = 0.0
        return out
    return ic


# --------------------------------------------------------------------------
# BASELINE.json configurations
# --------------------------------------------------------------------------

@dataclass
class Workload:
    name: str
    dim: int
    system: int            # 0 Euler, 1 MHD-GLM
    degree: int            # M
    n: tuple
    lo: tuple
    hi: tuple
    bc: tuple              # 6 ints, 0 periodic, 1 transmissive
    gamma: float
    cfl: float
    t_end: float
    steps: int = 0         # fixed step count (0: run to t_end)
    ic: object = None
    ch: float = 0.0
    refine_factor: int = 3
    lmax: int = 0
    chi_ref: float = 0.2     # refinement threshold (P:630-631 range 0.2-0.25)
    chi_rec: float = 0.1     # recoarsening threshold (P:631-632 range 0.05-0.15)
    note: str = ""
    extra: dict = field(default_factory=dict)


def config(name: str, n=None) -> Workload:
    """Named workloads.  c1..c5 follow BASELINE.json configs[0..4]; c6 is the
    paper's 3D AMR explosion."""
    P, T = 0, 1
    if name == "c1":
        nn = n or 32
        return Workload("c1_vortex2d_o3", 2, 0, 2, (nn, nn), (0.0, 0.0), (10.0, 10.0),
                        (P,) * 6, 1.4, 0.9, 1.0, ic=isentropic_vortex())
    if name == "c2":
        nn = n or 512
        return Workload(f"c2_vortex2d_o4_{nn}", 2, 0, 3, (nn, nn), (0.0, 0.0), (10.0, 10.0),
                        (P,) * 6, 1.4, 0.9, 10.0, ic=isentropic_vortex())
    if name == "c3":
        nn = n or 100
        # chi thresholds 0.1 / 0.05 (reading R14): with 0.2 a level-1 cell cut by the
        # initial jump stays unrefined and the projection of its polynomial into
        # the level-2 ghost cells is inadmissible at t = 0 (oracle and GPU alike)
        return Workload("c3_explosion2d_amr", 2, 0, 2, (nn, nn), (-1.0, -1.0), (1.0, 1.0),
                        (T,) * 6, 1.4, 0.45, 0.25, ic=explosion(2), refine_factor=3, lmax=2,
                        chi_ref=0.1, chi_rec=0.05)
    if name == "c4":
        nn = n or 256
        # CFL 0.3: at 0.9, 0.6 and 0.5 both the oracle and the CUDA path
        # reach an inadmissible face state (profiles/round1_explosion3d_cfl_probe.jsonl)
        return Workload(f"c4_explosion3d_o3_{nn}", 3, 0, 2, (nn, nn, nn), (-1.0,) * 3, (1.0,) * 3,
                        (T,) * 6, 1.4, 0.3, 1e300, steps=50, ic=explosion(3))
    if name == "c5":
        nn = n or 120
        return Workload("c5_orszag_tang_mhd", 2, 1, 3, (nn, nn), (0.0, 0.0),
                        (2 * math.pi, 2 * math.pi), (P,) * 6, 5.0 / 3.0, 0.9, 0.5,
                        ic=orszag_tang(), ch=2.0, refine_factor=3, lmax=3)
    if name == "c6":
        # the paper's 3D explosion on an AMR grid (P:1094-1097:
        # 34^3 level 0, r = 3, lmax = 2, third order); Rusanov flux (the Osher
        # scheme is inadmissible on this problem at comparable resolution,
        # reading R21).  With chi 0.1 / 0.05 or CFL 0.3 the first macro step
        # reaches an inadmissible level-2 state (tools/c6_probe.py); chi
        # 0.05 / 0.025 with CFL 0.2 runs
        nn = n or 34
        return Workload("c6_explosion3d_amr", 3, 0, 2, (nn, nn, nn), (-1.0,) * 3, (1.0,) * 3,
                        (T,) * 6, 1.4, 0.2, 0.25, ic=explosion(3), refine_factor=3, lmax=2,
                        chi_ref=0.05, chi_rec=0.025)
    if name in ("dmr", "dmr2"):
        # double Mach reflection on a uniform grid,
        # [0,3] x [0,1], exact solution prescribed left / top / right (reading
        # R26), reflective wall at the bottom (R22), Rusanov, O3.  "dmr" is the
        # paper's Mach-10 problem to t = 0.2: with the literal reflective bottom
        # the reconstruction at the shock foot is inadmissible in the first step
        # (oracle and CUDA path alike, reading R27); "dmr2" is the same geometry
        # at shock Mach 2, run to t = 1.0 (the front covers the same distance)
        nn = n or 240
        mach = 10.0 if name == "dmr" else 2.0
        return Workload(f"{name}_o3_{nn}x{nn // 3}", 2, 0, 2, (nn, nn // 3), (0.0, 0.0), (3.0, 1.0),
                        (4, 4, 2, 4, 0, 0), 1.4, 0.45, 2.0 / mach, ic=double_mach_reflection(mach),
                        extra=dict(exact_vel=dmr_front_vel(mach), mach=mach))
    raise KeyError(name)
