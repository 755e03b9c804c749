"""Partitioned (multi-rank) uniform path on the GPU, bitwise against one rank.

The n ranks of a Cartesian partition run as n contexts in this process on the
one GPU (ader_debug_group_*): the same pack / unpack kernels, halo plans,
boundary masks and redundant ghost-layer predictor as the NCCL path, with the
slabs NCCL would carry copied device to device and the CFL max taken on the
host.  Every cell's arithmetic is local, so any partition must reproduce the
one-rank state bit for bit.  Only the NCCL calls themselves
are not exercised here (one GPU per box).

AMR: every rank mirrors the tree, computes the cells whose level-0 ancestor
lies within the band of its level-0 block, and the owners' new averages are
copied into the other ranks' bands after every level update; the indicator is
merged over the owners.  The union of the ranks' subtrees must equal the
one-rank tree bit for bit (cell sets, statuses and averages).
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
    "box2d_walls_x4": (dict(dim=2, degree=2, n0=(20, 18), lo=(0, 0), hi=(1, 1), bc=(2,) * 6, cfl=0.45),
                       W.random_smooth(2, seed=3585, amp=0.2), 4, 5),
    "inflow3d_x4": (dict(dim=3, degree=2, n0=(12, 10, 9), lo=(0,) * 3, hi=(1,) * 3, bc=(3, 1, 0, 0, 3, 1), cfl=0.3),
                    W.random_smooth(3, seed=1212, amp=0.08), 4, 3),
    # time-dependent exact boundaries (R26): the DMR geometry at Mach 2, and a
    # traveling wave leaving / entering through exact sides in 3D
    "dmr2_exact_x3": (dict(dim=2, degree=2, n0=(48, 16), lo=(0, 0), hi=(3, 1), bc=(4, 4, 2, 4, 0, 0), cfl=0.45,
                           exact_vel=W.dmr_front_vel(2.0)), W.double_mach_reflection(2.0), 3, 6),
    "traveling3d_exact_x4": (dict(dim=3, degree=2, n0=(12, 10, 9), lo=(0,) * 3, hi=(1,) * 3, bc=(4,) * 6, cfl=0.5,
                                  exact_vel=(0.8, 0.35, -0.2)),
                             W.entropy_wave(3, amp=0.2, v=(0.8, 0.35, -0.2)), 4, 4),
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


AMR_CASES = {
    "explosion2d_l2_x4": (dict(dim=2, degree=2, n0=(30, 30), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=2, cfl=0.45,
                               chi_ref=0.1, chi_rec=0.05), W.explosion(2), 4, 4),
    "explosion2d_l2_osher_x2": (dict(dim=2, degree=2, n0=(24, 20), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=2,
                                     cfl=0.45, chi_ref=0.1, chi_rec=0.05, flux=1), W.explosion(2), 2, 3),
    "vortex2d_M3_l1_periodic_x3": (dict(dim=2, degree=3, n0=(30, 24), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, lmax=1,
                                        cfl=0.9, chi_ref=0.01, chi_rec=0.005), W.isentropic_vortex(), 3, 3),
    "ot_mhd_M3_l1_x4": (dict(dim=2, degree=3, n0=(32, 32), lo=(0, 0), hi=(2 * math.pi, 2 * math.pi), bc=(0,) * 6,
                             lmax=1, system=1, gamma=5 / 3, ch=2.0, cfl=0.45, chi_ref=0.02, chi_rec=0.01),
                        W.orszag_tang(), 4, 2),
    "explosion3d_l1_x2": (dict(dim=3, degree=2, n0=(16, 10, 10), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, lmax=1,
                               cfl=0.3), W.explosion(3), 2, 2),
    "explosion2d_l2_x8_long": (dict(dim=2, degree=2, n0=(40, 32), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=2,
                                    cfl=0.45, chi_ref=0.1, chi_rec=0.05), W.explosion(2), 8, 12),
    "quadrant_walls_l2_x4": (dict(dim=2, degree=2, n0=(24, 24), lo=(0, 0), hi=(1, 1), bc=(2, 1, 2, 1, 0, 0), lmax=2,
                                  cfl=0.45, chi_ref=0.1, chi_rec=0.05), W.explosion(2), 4, 5),
}


def _key_sorted(cells, nv):
    rows = sorted(((c.level, c.idx[2], c.idx[1], c.idx[0], c.status, tuple(c.u[:nv])) for c in cells))
    return rows


@pytest.mark.parametrize("name", list(AMR_CASES))
def test_amr_partition_reproduces_one_rank_bitwise(name):
    kw, ic, nr, steps = AMR_CASES[name]
    nv = 9 if kw.get("system", 0) == 1 else kw["dim"] + 2
    one = ader.Solver(ader.make_config(device=0, adapt_every=1, **kw))
    one.set_initial(ic)
    grp = ader.LoopbackGroup(ader.make_config(device=0, adapt_every=1, **kw), nr)
    grp.set_initial(ic)
    a, b = _key_sorted(one.get_cells(), nv), _key_sorted(grp.get_cells(), nv)
    assert a == b                                      # initial hierarchy
    r1 = one.step(1e300, steps)
    reps = grp.step(1e300, steps)
    assert all(r.dt0 == r1.dt0 for r in reps)
    assert sum(r.cell_updates for r in reps) == r1.cell_updates
    a, b = _key_sorted(one.get_cells(), nv), _key_sorted(grp.get_cells(), nv)
    assert len(a) == len(b)
    assert [x[:5] for x in a] == [x[:5] for x in b]    # cell sets and statuses
    bad = [(x, y) for x, y in zip(a, b) if x != y]
    assert not bad, bad[:3]                            # averages bit for bit
    grp.close()
    one.close()


# Dynamic load balancing (reading R24): after every adapt the level-0 blocks
# are re-cut by recursive coordinate bisection on the subtrees' local steps and
# the averages move to their new owners.  The partition must still reproduce
# one rank bit for bit, and the owned local steps must end up more even than
# with the static blocks (the blast sits in one corner / one end).
LB_CASES = {
    "quadrant_walls_l2_x4": (dict(dim=2, degree=2, n0=(24, 24), lo=(0, 0), hi=(1, 1), bc=(2, 1, 2, 1, 0, 0), lmax=2,
                                  cfl=0.45, chi_ref=0.1, chi_rec=0.05), W.explosion(2), 4, 5),
    "offcentre_l1_x3": (dict(dim=2, degree=2, n0=(48, 16), lo=(-1, -1), hi=(5, 1), bc=(1,) * 6, lmax=1, cfl=0.45,
                             chi_ref=0.1, chi_rec=0.05), W.explosion(2), 3, 4),
    "offcentre3d_l1_x2": (dict(dim=3, degree=2, n0=(20, 8, 8), lo=(-1, -1, -1), hi=(4, 1, 1), bc=(1,) * 6, lmax=1,
                               cfl=0.3), W.explosion(3), 2, 2),
    # periodic wrap of the compute band around re-cut (non-grid) blocks
    "vortex_periodic_M3_l1_x4": (dict(dim=2, degree=3, n0=(24, 24), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, lmax=1,
                                      cfl=0.9, chi_ref=0.01, chi_rec=0.005), W.isentropic_vortex(center=(2.0, 2.5)),
                                 4, 3),
}


@pytest.mark.parametrize("name", list(LB_CASES))
def test_dynamic_load_balance_keeps_bitwise_parity_and_evens_the_load(name):
    kw, ic, nr, steps = LB_CASES[name]
    nv = kw["dim"] + 2
    one = ader.Solver(ader.make_config(device=0, adapt_every=1, **kw))
    one.set_initial(ic)
    r1 = one.step(1e300, steps)
    a = _key_sorted(one.get_cells(), nv)
    one.close()
    imb = {}
    for lb in (0, 1):
        grp = ader.LoopbackGroup(ader.make_config(device=0, adapt_every=1, load_balance=lb, **kw), nr)
        grp.set_initial(ic)
        reps = grp.step(1e300, steps)
        assert all(r.dt0 == r1.dt0 for r in reps)
        assert sum(r.cell_updates for r in reps) == r1.cell_updates
        b = _key_sorted(grp.get_cells(), nv)
        assert len(a) == len(b)
        bad = [(x, y) for x, y in zip(a, b) if x != y]
        assert not bad, (lb, bad[:3])
        loads = [r.cell_updates for r in reps]
        imb[lb] = max(loads) * nr / sum(loads)
        if lb == 0:
            assert all(r.rebalances == 0 for r in reps)
        grp.close()
    print(f"{name}: owned local-step imbalance static {imb[0]:.3f} -> dynamic {imb[1]:.3f}")
    assert imb[1] < imb[0] and imb[1] < 1.3, imb


# Reading R28: the multi-rank compute sets follow the dependencies of the owned
# updates instead of a 2(M+1) level-0 band on every level.  The partition must
# still reproduce one rank bit for bit, and the computed cells (local steps of
# all ranks' predictors) stay within 1.2x the owned ones at 8 ranks.
@pytest.mark.parametrize("name", ["explosion2d_l2_x8_long"])
def test_amr_dependency_sets_cut_redundant_work(name, monkeypatch):
    kw, ic, nr, steps = AMR_CASES[name]
    nv = kw["dim"] + 2
    one = ader.Solver(ader.make_config(device=0, adapt_every=1, **kw))
    one.set_initial(ic)
    r1 = one.step(1e300, steps)
    a = _key_sorted(one.get_cells(), nv)
    one.close()
    ratio = {}
    for band in ("1", "0"):
        monkeypatch.setenv("ADER_AMR_BAND", band)
        grp = ader.LoopbackGroup(ader.make_config(device=0, adapt_every=1, **kw), nr)
        grp.set_initial(ic)
        reps = grp.step(1e300, steps)
        assert sum(r.cell_updates for r in reps) == r1.cell_updates
        assert _key_sorted(grp.get_cells(), nv) == a
        ratio[band] = sum(r.pred_cells for r in reps) / sum(r.cell_updates for r in reps)
        grp.close()
    print(f"{name}: computed / owned local steps band {ratio['1']:.3f} -> dependency sets {ratio['0']:.3f}")
    assert ratio["0"] < ratio["1"] and ratio["0"] <= 1.2, ratio
