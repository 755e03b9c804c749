"""GPU: the predictor's x contraction on the FP64 tensor cores (dmma_x, 2D
M = 3, the default) gives bitwise the q, states, AMR cell sets and sweep
counts of the shared-memory contraction (ADER_PRED_DMMA=0): the MMA
accumulates in k order like the scalar FMA chain of eqn.stdg.final's nodal
form.  The variant is chosen once per process, so each side runs
tools/pred_ab.py in its own subprocess (uniform Euler with and without the
R25 guess, walls, Orszag-Tang MHD, AMR Euler and MHD)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dmma_x_contraction_bitwise_equals_shared_memory_form(tmp_path):
    out = {}
    for flag in ("0", "1"):
        env = dict(os.environ, ADER_PRED_DMMA=flag)
        path = tmp_path / f"p{flag}.npz"
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pred_ab.py"), "save", str(path)], env=env,
                       check=True, timeout=600)
        out[flag] = np.load(path)
    assert sorted(out["0"].files) == sorted(out["1"].files)
    for k in out["0"].files:
        assert np.array_equal(out["0"][k], out["1"][k]), k
