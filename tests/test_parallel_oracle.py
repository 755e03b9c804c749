"""The multi-process oracle runner (tests/parallel_oracle.py) reproduces the
serial oracle bit for bit (no GPU)."""
import numpy as np
import pytest

import oracle as O
from paper_1212_3585_b200 import workloads as W
from tests import parallel_oracle as PO


@pytest.mark.parametrize("kw,ic,steps", [
    (dict(dim=2, degree=2, n=(18, 16), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9), W.isentropic_vortex(), 3),
    (dict(dim=3, degree=2, n=(5, 4, 6), lo=(-1,) * 3, hi=(1,) * 3, bc=(1, 2, 1, 1, 2, 1), cfl=0.3), W.explosion(3), 2),
])
def test_parallel_runner_is_bitwise_serial(kw, ic, steps):
    o = O.Oracle(**kw)
    o.set_initial(ic)
    o.step(1e300, steps)
    u, n, t = PO.run(kw, ic, max_steps=steps, nproc=3)
    assert n == steps and t == o.t
    assert np.array_equal(u, o.get_cells())
