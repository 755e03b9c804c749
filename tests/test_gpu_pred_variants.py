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


def _ab(tool, tmp_path, var, flags, extra_env=None):
    out = {}
    for flag in flags:
        env = dict(os.environ, **{var: flag}, **(extra_env or {}))
        path = tmp_path / f"{var}_{flag}.npz"
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool), "save", str(path)], env=env, check=True,
                       timeout=900, stdout=subprocess.DEVNULL)
        out[flag] = np.load(path)
    a, b = out[flags[0]], out[flags[1]]
    assert sorted(a.files) == sorted(b.files)
    return a, b


def test_flat_cell_first_sweep_bitwise_equals_general_path(tmp_path):
    """The predictor's flat-cell first sweep (every node of the warp's cells carries the same w: each lane
    contracts its own f*, eqn.stdg.final P:463-474 with the time-constant guess R3) gives bitwise the q, F and
    states of the shared-memory contraction (ADER_PRED_FLAT=0) on explosions with constant regions (3D M = 2,
    walls, Osher), the vortex and MHD."""
    a, b = _ab("flux_ab.py", tmp_path, "ADER_PRED_FLAT", ("0", "1"))
    for k in a.files:
        if not k.endswith("_flatcount"):
            assert np.array_equal(a[k], b[k]), k


def test_flat_cells_without_q_block_give_bitwise_the_same_fluxes_and_states(tmp_path):
    """3D M = 2, opt-in (ADER_PRED_FLAT_SKIP=1): a flat cell that converges in the first sweep gets a flag
    instead of its q_h block and the face-flux kernel rebuilds q_h = w - Tsum[s] G(node) from w (the
    predictor's own flat first sweep, eqn.stdg.final P:463-474 with guess R3; traces of flux:F/G/H
    P:158-172).  F, q and the states after a few steps are bitwise those of the default (every block written
    and read), on explosions with constant regions (transmissive sides, walls, Osher) as on the vortex and
    MHD cases without flat cells; the report counts the flat cells either way."""
    a, b = _ab("flux_ab.py", tmp_path, "ADER_PRED_FLAT_SKIP", ("0", "1"))
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
    for name in ("c4_expl3d_24", "expl3d_walls", "osher3d"):
        assert 0 < b[name + "_flatcount"][0] < b[name + "_flatcount"][1]
    assert b["vortex_m2_flatcount"][0] == 0


def test_amr_sibling_patch_weno_bitwise_equals_per_cell_box(tmp_path):
    """AMR reconstruction (P:276-322 on the cell-by-cell tree): sweeping the window of a mother's children
    once (k_amr_weno_patch) solves the same 1D problems as every child's own (2M+1)^d box
    (ADER_AMR_WENO_PATCH=0): cell sets, averages and update counts bitwise equal after several macro steps
    (2D M = 2 lmax = 2, walls, 2D M = 3, MHD lmax = 2, 3D lmax = 2)."""
    a, b = _ab("amr_weno_ab.py", tmp_path, "ADER_AMR_WENO_PATCH", ("0", "1"))
    for k in a.files:
        assert a[k].shape == b[k].shape and np.array_equal(a[k], b[k]), k


def test_rotation_shuffle_flux_matches_gather_flux(tmp_path):
    """The face flux from coalesced block loads and warp-shuffle line sums (flux_rot.cu, ADER_FLUX_ROT=1)
    forms the traces of flux:F/G/H with their N products in a rotated order and sums the points
    in node order: F, q and the states after a few steps agree with the default kernel to rounding."""
    a, b = _ab("flux_ab.py", tmp_path, "ADER_FLUX_ROT", ("0", "1"))
    for k in a.files:
        if k.endswith("_flatcount"):
            continue
        d = np.abs(a[k] - b[k]).max()
        assert d <= 1e-13 * max(np.abs(a[k]).max(), 1e-300), (k, d)


def test_x_run_flux_bitwise_equals_cell_flux(tmp_path):
    """3D M = 2 Euler/Rusanov default: the face-flux kernel that walks runs of 8 cells along x and carries the
    xi = 1 trace (flux:F/G/H P:158-172, eqn.rusanov) gives bitwise the F, q and states of
    k_face_flux_cells (ADER_FLUX_RUNS=0), on explosions with transmissive sides and walls."""
    a, b = _ab("flux_ab.py", tmp_path, "ADER_FLUX_RUNS", ("0", "5"))
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
