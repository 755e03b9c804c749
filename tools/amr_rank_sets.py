"""Multi-rank AMR compute sets (reading R28) against the round-1 uniform band:
for a loopback partition of W ranks (one process, one GPU) run a few macro
steps of a workload and report computed / owned = sum over ranks of the
predicted cells over sum of the owned local steps (both in local steps), for
ADER_AMR_BAND=1 (band 2(M+1) level-0 cells on every level) and the default
dependency sets; check that the partition reproduces one rank bit for bit.

  python tools/amr_rank_sets.py [--w 8] [--steps 3] c3 c5 c6 ...
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_3585_b200 import ader  # noqa: E402
from paper_1212_3585_b200 import workloads as W  # noqa: E402


def cfg_of(wl, **kw):
    return ader.make_config(dim=wl.dim, degree=wl.degree, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, system=wl.system,
                            gamma=wl.gamma, ch=wl.ch, cfl=wl.cfl, lmax=wl.lmax, refine_factor=wl.refine_factor,
                            chi_ref=wl.chi_ref, chi_rec=wl.chi_rec, adapt_every=1, device=0, **kw)


def key(cells, nv):
    return sorted((c.level, c.idx[2], c.idx[1], c.idx[0], c.status, tuple(c.u[:nv])) for c in cells)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--w", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--no-one", action="store_true", help="skip the one-rank bitwise reference")
    a = ap.parse_args()
    for name in a.names:
        wl = W.config(name, a.n or None)
        nv = 9 if wl.system == 1 else wl.dim + 2
        ref = None
        if not a.no_one:
            one = ader.Solver(cfg_of(wl))
            one.set_initial(wl.ic)
            r1 = one.step(1e300, a.steps)
            ref = key(one.get_cells(), nv)
            one.close()
        out = {"workload": wl.name, "ranks": a.w, "macro_steps": a.steps}
        for mode in ("band", "deps"):
            os.environ["ADER_AMR_BAND"] = "1" if mode == "band" else "0"
            g = ader.LoopbackGroup(cfg_of(wl), a.w)
            g.set_initial(wl.ic)
            reps = g.step(1e300, a.steps)
            owned = sum(r.cell_updates for r in reps)
            comp = sum(r.pred_cells for r in reps)
            per = [r.pred_cells / max(1, r.cell_updates) for r in reps]
            same = None
            if ref is not None:
                same = key(g.get_cells(), nv) == ref and owned == r1.cell_updates
            out[mode] = {"computed_over_owned": comp / owned, "max_rank_ratio": max(per), "owned_updates": owned,
                         "bitwise_one_rank": same}
            g.close()
        os.environ.pop("ADER_AMR_BAND", None)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
