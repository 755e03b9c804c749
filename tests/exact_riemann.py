"""Exact Riemann solver for the 1D Euler equations (ideal gas).

Textbook construction (pressure function + Newton iteration for p*, then
sampling of the self-similar solution), written here as an independent check
of the oracle: the paper itself compares against reference solutions it does
not ship, so the shock-tube pin uses this closed-form solution.
"""
from __future__ import annotations

import math

import numpy as np


def _f(p, rho, pk, ck, g):
    if p > pk:   # shock
        A = 2.0 / ((g + 1.0) * rho)
        B = (g - 1.0) / (g + 1.0) * pk
        s = math.sqrt(A / (p + B))
        return (p - pk) * s, s * (1.0 - 0.5 * (p - pk) / (B + p))
    pr = p / pk   # rarefaction
    return (2.0 * ck / (g - 1.0)) * (pr ** ((g - 1.0) / (2.0 * g)) - 1.0), \
        1.0 / (rho * ck) * pr ** (-(g + 1.0) / (2.0 * g))


def star_state(WL, WR, g=1.4):
    rl, ul, pl = WL
    rr, ur, pr = WR
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    p = max(1e-10, 0.5 * (pl + pr) - 0.125 * (ur - ul) * (rl + rr) * (cl + cr))
    for _ in range(100):
        fl, dfl = _f(p, rl, pl, cl, g)
        fr, dfr = _f(p, rr, pr, cr, g)
        dp = (fl + fr + ur - ul) / (dfl + dfr)
        pn = max(1e-12, p - dp)
        if abs(pn - p) < 1e-14 * (pn + p):
            p = pn
            break
        p = pn
    fl, _ = _f(p, rl, pl, cl, g)
    fr, _ = _f(p, rr, pr, cr, g)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def sample(WL, WR, s, g=1.4):
    """Primitive (rho, u, p) of the exact solution at x/t = s (array)."""
    rl, ul, pl = WL
    rr, ur, pr = WR
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    ps, us = star_state(WL, WR, g)
    s = np.asarray(s, dtype=np.float64)
    out = np.zeros((s.size, 3))
    for i, si in enumerate(s.ravel()):
        if si <= us:   # left of contact
            if ps > pl:
                rs = rl * ((ps / pl + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pl + 1))
                S = ul - cl * math.sqrt((g + 1) / (2 * g) * ps / pl + (g - 1) / (2 * g))
                out[i] = (rl, ul, pl) if si <= S else (rs, us, ps)
            else:
                rs = rl * (ps / pl) ** (1 / g)
                cs = cl * (ps / pl) ** ((g - 1) / (2 * g))
                sh, st = ul - cl, us - cs
                if si <= sh:
                    out[i] = (rl, ul, pl)
                elif si >= st:
                    out[i] = (rs, us, ps)
                else:
                    u = 2 / (g + 1) * (cl + (g - 1) / 2 * ul + si)
                    c = 2 / (g + 1) * (cl + (g - 1) / 2 * (ul - si))
                    r = rl * (c / cl) ** (2 / (g - 1))
                    out[i] = (r, u, pl * (c / cl) ** (2 * g / (g - 1)))
        else:
            if ps > pr:
                rs = rr * ((ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1))
                S = ur + cr * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
                out[i] = (rr, ur, pr) if si >= S else (rs, us, ps)
            else:
                rs = rr * (ps / pr) ** (1 / g)
                cs = cr * (ps / pr) ** ((g - 1) / (2 * g))
                sh, st = ur + cr, us + cs
                if si >= sh:
                    out[i] = (rr, ur, pr)
                elif si <= st:
                    out[i] = (rs, us, ps)
                else:
                    u = 2 / (g + 1) * (-cr + (g - 1) / 2 * ur + si)
                    c = 2 / (g + 1) * (cr - (g - 1) / 2 * (ur - si))
                    r = rr * (c / cr) ** (2 / (g - 1))
                    out[i] = (r, u, pr * (c / cr) ** (2 * g / (g - 1)))
    return out


def cell_average_density(WL, WR, x0, t, edges, g=1.4, sub=64):
    """Exact cell averages of rho on cells [edges[i], edges[i+1]] (midpoint sub-sampling)."""
    edges = np.asarray(edges, dtype=np.float64)
    out = np.zeros(len(edges) - 1)
    for i in range(len(edges) - 1):
        xs = edges[i] + (np.arange(sub) + 0.5) / sub * (edges[i + 1] - edges[i])
        out[i] = sample(WL, WR, (xs - x0) / t, g)[:, 0].mean()
    return out
