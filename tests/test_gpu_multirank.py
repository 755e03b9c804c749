"""Partitioned (multi-rank) uniform path on the GPU, bitwise against one rank.

The n ranks of a Cartesian partition run as n contexts in this process on the
one GPU (ader_debug_group_*): the same pack / unpack kernels, halo plans,
boundary masks and redundant ghost-layer predictor as the NCCL path, with the
slabs NCCL would carry copied device to device and the CFL max taken on the
host.  Every cell's arithmetic is local, so any partition must reproduce the
one-rank state bit for bit.  Only the NCCL calls themselves
are not exercised here (one GPU per box).
"""
import math

import numpy as np
import pytest

from paper_1212_3585_b200 import ader
from paper_1212_3585_b200 import workloads as W

pytestmark = pytest.mark.gpu

CASES = {
    "vortex2d_M3_periodic_x2": (dict(dim=2, degree=3, n0=(24, 20), lo=(0, 0), hi=(10, 10), bc=(0,) * 6),
                                W.isentropic_vortex(), 2, 6),
    "vortex2d_M2_periodic_x4": (dict(dim=2, degree=2, n0=(26, 22), lo=(0, 0), hi=(10, 10), bc=(0,) * 6),
                                W.isentropic_vortex(), 4, 6),
    "explosion2d_M2_transmissive_x3": (dict(dim=2, degree=2, n0=(30, 17), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6),
                                       W.explosion(2), 3, 5),
    "explosion2d_osher_x4": (dict(dim=2, degree=2, n0=(24, 24), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, flux=1),
                             W.explosion(2), 4, 5),
    "explosion3d_M2_transmissive_x8": (dict(dim=3, degree=2, n0=(12, 14, 10), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6,
                                            cfl=0.3), W.explosion(3), 8, 4),
    "random3d_M2_periodic_x6": (dict(dim=3, degree=2, n0=(12, 9, 13), lo=(0,) * 3, hi=(1,) * 3, bc=(0,) * 6),
                                W.random_smooth(3, seed=1212, amp=0.08), 6, 3),
    "ot_mhd_M3_periodic_x2": (dict(dim=2, degree=3, n0=(16, 18), lo=(0, 0), hi=(2 * math.pi, 2 * math.pi),
                                   bc=(0,) * 6, system=1, gamma=5 / 3, ch=2.0), W.orszag_tang(), 2, 4),
}


@pytest.mark.parametrize("name", list(CASES))
def test_partition_reproduces_one_rank_bitwise(name):
    kw, ic, nr, steps = CASES[name]
    cfg1 = ader.make_config(device=0, **kw)
    one = ader.Solver(cfg1)
    one.set_initial(ic)
    r1 = one.step(1e300, steps)
    d = kw["dim"]
    n0 = list(kw["n0"]) + [1] * (3 - d)
    u1 = one.get_state().reshape(n0[2], n0[1], n0[0], -1)

    grp = ader.LoopbackGroup(ader.make_config(device=0, **kw), nr)
    grid = set(tuple(p.dims) for p in grp.parts)
    assert len(grid) == 1 and np.prod(next(iter(grid))) == nr
    grp.set_initial(ic)
    reps = grp.step(1e300, steps)
    assert all(r.macro_steps == steps for r in reps)
    assert all(r.dt0 == r1.dt0 for r in reps)          # the CFL max over ranks is exact
    assert sum(r.cell_updates for r in reps) == r1.cell_updates
    ug = grp.gather()
    assert np.array_equal(ug, u1), np.abs(ug - u1).max()
    grp.close()
    one.close()


def test_group_rejects_thin_blocks_and_plain_step():
    # blocks thinner than the ghost layer M+1 are a configuration error
    cfg = ader.make_config(dim=2, degree=2, n0=(4, 4), lo=(0, 0), hi=(1, 1), bc=(0,) * 6, device=0)
    with pytest.raises(ader.AderError):
        ader.LoopbackGroup(cfg, 4)
    cfg = ader.make_config(dim=2, degree=2, n0=(16, 16), lo=(0, 0), hi=(1, 1), bc=(0,) * 6, device=0)
    grp = ader.LoopbackGroup(cfg, 2)
    st = ader.lib().ader_step(grp.ptrs[0], 1e300, 1, None)
    assert st == 1
    grp.close()
