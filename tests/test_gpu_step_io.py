"""ader_step_io (the e2e path: state in from the host — in slabs along the last
axis overlapped with the ghost fill / WENO sweeps of the slabs already in —
one macro step, state out with the copy-out overlapped by the slab-wise face
fluxes / update) gives bitwise the state of ader_set_cells + ader_step(1) +
ader_get_state."""
import numpy as np
import pytest
import torch

from paper_1212_3585_b200 import ader
from paper_1212_3585_b200 import workloads as W

pytestmark = pytest.mark.gpu

CASES = {
    "vortex2d_M3_periodic": (dict(dim=2, degree=3, n0=(70, 66), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                             W.isentropic_vortex()),
    "explosion3d_transmissive": (dict(dim=3, degree=2, n0=(20, 18, 37), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6,
                                      cfl=0.3), W.explosion(3)),
    "explosion3d_walls": (dict(dim=3, degree=2, n0=(12, 12, 9), lo=(0,) * 3, hi=(1,) * 3, bc=(2, 1, 2, 1, 2, 1),
                               cfl=0.3), W.explosion(3)),
    "ot_mhd_M3": (dict(dim=2, degree=3, n0=(40, 17), lo=(0, 0), hi=(2 * np.pi, 2 * np.pi), bc=(0,) * 6, system=1,
                       gamma=5 / 3, ch=2.0, cfl=0.5), W.orszag_tang()),
    # slab-pipelined copy-in (n along the last axis >= 16): walls and periodic in 3D
    "explosion3d_walls_tall": (dict(dim=3, degree=2, n0=(10, 9, 33), lo=(0,) * 3, hi=(1,) * 3, bc=(2, 1, 2, 1, 2, 1),
                                    cfl=0.3), W.explosion(3)),
    "random3d_periodic": (dict(dim=3, degree=2, n0=(12, 11, 24), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6, cfl=0.3),
                          W.random_smooth(3)),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("pipeline", ["0", "1"])
def test_step_io_equals_set_step_get(name, fuse, pipeline, monkeypatch):
    monkeypatch.setenv("ADER_STEP_IO_PIPELINE", pipeline)
    kw, ic = CASES[name]
    a = ader.Solver(ader.make_config(device=0, fuse_pred_flux=fuse, **kw))
    b = ader.Solver(ader.make_config(device=0, fuse_pred_flux=fuse, **kw))
    a.set_initial(ic)
    b.set_initial(ic)
    host = torch.empty((a.ncells, a.nv), dtype=torch.float64, pin_memory=True)
    a.get_state_ptr(host.data_ptr())
    for _ in range(3):
        ra = a.step_io(host.data_ptr(), host.data_ptr())
        rb = b.step(1e300, 1)
        ub = b.get_state()
        assert ra.dt0 == rb.dt0 and ra.macro_steps == 1
        assert np.array_equal(host.numpy(), ub)
        assert np.array_equal(a.get_state(), ub)
    # a state from the host that differs from the device's (set_cells semantics)
    host.numpy()[:] = ub[::-1] if kw.get("system", 0) == 0 and kw["bc"][0] == 0 else ub
    b.set_cells(host.numpy().copy())
    a.step_io(host.data_ptr(), host.data_ptr())
    b.step(1e300, 1)
    assert np.array_equal(host.numpy(), b.get_state())
    a.close()
    b.close()


# Uniform steps replay as one CUDA graph per macro step (profiling off, one
# rank): bitwise the same states and the same launch accounting as the
# directly enqueued kernels (ADER_NO_GRAPHS=1), also across a change of t_end
# (the graph is re-captured: k_step_dt clips against it).
@pytest.mark.parametrize("name", ["vortex2d_M3_periodic", "explosion3d_walls"])
def test_graph_replay_equals_direct_launches(name, monkeypatch):
    kw, ic = CASES[name]
    out = {}
    for off in ("0", "1"):
        monkeypatch.setenv("ADER_NO_GRAPHS", off)
        s = ader.Solver(ader.make_config(device=0, **kw))
        s.set_initial(ic)
        l0 = s.launch_count()
        r1 = s.step(1e300, 7)
        r2 = s.step(r1.t + 2.5 * r1.dt0, 10)   # ends inside the third step: dt clipped
        out[off] = (s.get_state(), s.launch_count() - l0, r1.t, r2.t, r2.macro_steps)
        s.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert out["0"][1:] == out["1"][1:]
