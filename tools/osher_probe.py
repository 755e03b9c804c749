"""Probe: the 3D explosion (BASELINE config 4 grid) with the Osher flux — which
CFL keeps it admissible for 50 steps on the GPU, and does the oracle reach the
same inadmissible state from the GPU's last good state (sampled box around the
failing cell)?  Prints JSON lines."""
import json
import os
import re
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def solver(n, cfl):
    wl = W.config("c4", n)
    cfg = ader.make_config(dim=3, degree=2, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=cfl, device=0, flux=1)
    s = ader.Solver(cfg)
    s.set_initial(wl.ic)
    return wl, s


def run(n, cfl, steps):
    wl, s = solver(n, cfl)
    t0 = time.time()
    k = 0
    out = dict(n=n, cfl=cfl, ok=True)
    try:
        for k in range(steps):
            r = s.step(1e300, 1)
        out.update(steps=steps, t=r.t)
    except ader.AderError as e:
        out.update(ok=False, fail_step=k, err=str(e))
    out["wall"] = time.time() - t0
    s.close()
    print(json.dumps(out), flush=True)
    return out


def oracle_check(n, cfl, fail_step, err):
    """Replay to the step before the failure, hand that state to the oracle and
    advance a box around the failing cell with the same dt."""
    import oracle as O
    m = re.search(r"cell \((\d+),(\d+),(\d+)\)", err)
    cell = [int(x) for x in m.groups()]
    wl, s = solver(n, cfl)
    if fail_step:
        s.step(1e300, fail_step)
    u = s.get_state()
    o = O.Oracle(dim=3, degree=2, n=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=cfl, flux=O.OSHER)
    o.set_cells(u)
    dt = o.compute_dt()
    blo = [max(0, c - 2) for c in cell]
    bhi = [min(n, c + 3) for c in cell]
    try:
        out, _ = o.advance_box(dt, blo, bhi)
        res = dict(oracle="ok", dt=dt, box=[blo, bhi])
        # and the GPU's own step from the same state
        try:
            s.step(1e300, 1)
            res["gpu"] = "ok"
        except ader.AderError as e:
            res["gpu"] = str(e)
    except Exception as e:  # noqa: BLE001
        res = dict(oracle=f"error: {e}", dt=dt, box=[blo, bhi])
    s.close()
    print(json.dumps(dict(n=n, cfl=cfl, fail_step=fail_step, **res)), flush=True)


if __name__ == "__main__":
    first_fail = None
    for n, cfl in [(256, 0.3), (256, 0.25), (256, 0.2), (128, 0.3), (64, 0.3)]:
        r = run(n, cfl, 50)
        if not r["ok"] and first_fail is None:
            first_fail = (n, cfl, r["fail_step"], r["err"])
    if first_fail is not None:
        oracle_check(*first_fail)
