"""c6 probe: which (chi_ref, cfl) keeps the 3D AMR explosion admissible for the first macro steps."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1212_3585_b200 import ader, workloads as W  # noqa: E402
wl = W.config("c6")
for chi, cfl in [(0.05, 0.3), (0.1, 0.2), (0.05, 0.2)]:
    cfg = ader.make_config(dim=3, degree=2, n0=wl.n, lo=wl.lo, hi=wl.hi, bc=wl.bc, cfl=cfl, lmax=2, refine_factor=3,
                           chi_ref=chi, chi_rec=chi / 2, adapt_every=1, device=0)
    s = ader.Solver(cfg)
    t0 = time.time()
    s.set_initial(wl.ic)
    out = dict(chi_ref=chi, cfl=cfl, init_s=time.time() - t0, cells=len(s.get_cells()))
    try:
        t0 = time.time()
        r = s.step(1e300, 3)
        out.update(ok=True, steps=r.macro_steps, updates=r.cell_updates, wall=time.time() - t0, cells_after=len(s.get_cells()))
    except ader.AderError as e:
        out.update(ok=False, err=str(e)[:200])
    s.close()
    print(json.dumps(out), flush=True)
