"""Test helper: run the uniform-grid oracle for many steps on several host
processes.  TEST INFRASTRUCTURE ONLY (it calls oracle/).

A step of the oracle (orc_step) is: dt from the CFL rule on the whole state,
then orc_advance_box on the whole box.  Every cell's new average depends only
on the old state (its reconstruction / predictor / face fluxes use ghost
cells from the same old state), so splitting the box into z- (3D) or y-slabs
(2D) and calling orc_advance_box on each slab in its own process gives the
serial result bit for bit; dt is taken from one oracle holding the whole state,
clipped to t_end exactly as orc_step does.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

import oracle as O

_W = None   # per-process oracle


def _init(kw, ic_name, ic_args):
    global _W
    _W = O.Oracle(**kw)


def _advance(args):
    state, dt, blo, bhi = args
    _W.set_cells(state)
    out, rep = _W.advance_box(dt, blo, bhi)
    return out, rep.sweeps_total


def run(kw, ic, t_end=1e300, max_steps=1, nproc=None):
    """Oracle(**kw) from ic, advanced like Oracle.step(t_end, max_steps) on nproc
    processes.  Returns (cells [ncell][nv], steps, t)."""
    o = O.Oracle(**kw)
    o.set_initial(ic)
    n = list(kw["n"])
    d = kw["dim"]
    nproc = nproc or min(16, os.cpu_count() or 1)
    ax = d - 1
    nsl = max(1, min(nproc, n[ax]))
    cuts = np.linspace(0, n[ax], nsl + 1).astype(int)
    boxes = []
    for i in range(nsl):
        lo = [0, 0, 0]
        hi = list(n) + [1] * (3 - len(n))
        lo[ax], hi[ax] = int(cuts[i]), int(cuts[i + 1])
        boxes.append((lo, hi))
    ctx = mp.get_context("fork")
    u = o.get_cells()
    t, steps = 0.0, 0
    shape = [n[2], n[1], n[0]] if d == 3 else [n[1], n[0]]
    with ctx.Pool(nsl, initializer=_init, initargs=(kw, None, None)) as pool:
        while steps < max_steps and t < t_end:
            o.set_cells(u)
            dt = o.compute_dt()
            assert dt > 0 and np.isfinite(dt)
            if t + dt > t_end:
                dt = t_end - t
            res = pool.map(_advance, [(u, dt, lo, hi) for lo, hi in boxes])
            new = np.empty(shape + [u.shape[1]])
            for (lo, hi), (out, _) in zip(boxes, res):
                if d == 3:
                    new[lo[2]:hi[2]] = out.reshape(hi[2] - lo[2], n[1], n[0], -1)
                else:
                    new[lo[1]:hi[1]] = out.reshape(hi[1] - lo[1], n[0], -1)
            u = new.reshape(-1, u.shape[1])
            t += dt
            steps += 1
    return u, steps, t
