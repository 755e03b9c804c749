"""Host-only checks of the dynamic load balancer's partitioner (reading R24,
ader.h: ader_rcb_partition, the paper's future work P:809-810).

Recursive coordinate bisection is checked against what fixes it independently
of the code: the boxes tile the level-0 grid exactly once; uniform weights on a
power-of-two rank count give equal boxes; for two ranks the cut is the
brute-force best plane of the longest axis; and a concentrated load ends up
balanced where the static Cartesian blocks are not.
"""
import itertools

import numpy as np
import pytest

from paper_1212_3585_b200 import ader


def _owner_grid(boxes, n):
    own = -np.ones((n[2], n[1], n[0]), dtype=int)
    for p, (lo, hi) in enumerate(boxes):
        blk = own[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        assert (blk == -1).all(), "boxes overlap"
        assert blk.size > 0, "empty box"
        blk[...] = p
    return own


def _loads(boxes, w):
    return [int(w[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].sum()) for lo, hi in boxes]


@pytest.mark.parametrize("dim,n,world", [(2, (12, 9, 1), 3), (3, (8, 6, 10), 8), (2, (40, 32, 1), 7), (3, (5, 5, 5), 5),
                                         (2, (7, 30, 1), 2)])
def test_boxes_tile_the_grid(dim, n, world):
    rng = np.random.default_rng(1212)
    w = rng.integers(1, 50, size=(n[2], n[1], n[0]))
    boxes = ader.ader_rcb_partition(dim, n[:dim], w, world)
    own = _owner_grid(boxes, n)
    assert (own >= 0).all(), "cells left without an owner"


def test_uniform_weights_on_a_power_of_two_give_equal_boxes():
    n = (16, 16, 16)
    boxes = ader.ader_rcb_partition(3, n, np.ones((16, 16, 16), dtype=np.int64), 8)
    assert sorted(_loads(boxes, np.ones((16, 16, 16)))) == [512] * 8
    assert all(tuple(h[k] - l[k] for k in range(3)) == (8, 8, 8) for l, h in boxes)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_two_ranks_take_the_brute_force_best_plane(seed):
    rng = np.random.default_rng(3585 + seed)
    n = (int(rng.integers(4, 20)), int(rng.integers(4, 20)), 1)
    w = rng.integers(0, 100, size=(1, n[1], n[0]))
    w[0, 0, 0] += 1
    boxes = ader.ader_rcb_partition(2, n[:2], w, 2)
    ax = 0 if n[0] >= n[1] else 1
    prof = w[0].sum(axis=0) if ax == 0 else w[0].sum(axis=1)     # weight per plane of the cut axis
    tot = prof.sum()
    devs = [abs(2 * prof[:c].sum() - tot) for c in range(1, n[ax])]
    best = 1 + int(np.argmin(devs))     # first minimiser
    (lo0, hi0), (lo1, hi1) = boxes
    assert hi0[ax] == best and lo1[ax] == best
    assert lo0[ax] == 0 and hi1[ax] == n[ax]
    for k in range(2):
        if k != ax:
            assert (lo0[k], hi0[k], lo1[k], hi1[k]) == (0, n[k], 0, n[k])


def test_concentrated_load_is_balanced():
    # explosion-like load: a refined disc in one corner of a 40x32 grid, cost
    # 1 + 9 + 81 per refined cell (r = 3, two levels), against the static 2x2 blocks
    n = (40, 32, 1)
    y, x = np.mgrid[0:32, 0:40]
    w = np.where((x - 5) ** 2 + (y - 4) ** 2 < 100, 81, 1).astype(np.int64)[None]
    for world in (2, 3, 4, 8):
        boxes = ader.ader_rcb_partition(2, n[:2], w, world)
        loads = _loads(boxes, w)
        assert max(loads) * world / sum(loads) < 1.25, (world, loads)
    static = [((0, 0, 0), (20, 16, 1)), ((20, 0, 0), (40, 16, 1)), ((0, 16, 0), (20, 32, 1)), ((20, 16, 0), (40, 32, 1))]
    loads = _loads(static, w)
    assert max(loads) * 4 / sum(loads) > 3.0


def test_rejections():
    w = np.ones((1, 4, 3), dtype=np.int64)
    with pytest.raises(ader.AderError):
        ader.ader_rcb_partition(2, (3, 4), w, 5)            # no axis long enough for five ranks
    with pytest.raises(ader.AderError):
        ader.ader_rcb_partition(2, (3, 4), -w, 2)           # negative weight
    with pytest.raises(ValueError):
        ader.ader_rcb_partition(2, (3, 5), w, 2)            # wrong weight count


def test_every_rank_count_up_to_eight_on_a_small_3d_grid():
    rng = np.random.default_rng(7)
    n = (9, 8, 10)
    w = rng.integers(0, 5, size=(n[2], n[1], n[0]))
    for world in range(1, 9):
        boxes = ader.ader_rcb_partition(3, n, w, world)
        own = _owner_grid(boxes, n)
        assert (own >= 0).all()
        assert len(set(itertools.chain.from_iterable([own.ravel().tolist()]))) == world
