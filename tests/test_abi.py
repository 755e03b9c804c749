"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/ader.h declares, rejects bad configurations before touching the
device, and partitions level-0 blocks consistently (host-only logic)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1212_3585_b200 import ader

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ader.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ader_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ader.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(ader.EXPORTED)


def _cfg(**kw):
    base = dict(dim=2, degree=2, n0=(16, 16), lo=(0, 0), hi=(1, 1), bc=(0,) * 6)
    base.update(kw)
    return ader.make_config(**base)


@pytest.mark.parametrize("kw", [dict(dim=4), dict(degree=1), dict(degree=5), dict(n0=(0, 4)),
                                dict(world_size=9), dict(rank=2, world_size=2), dict(gamma=1.0),
                                dict(bc=(0, 1, 0, 0, 0, 0)), dict(dim=3, degree=3, n0=(8, 8, 8)),
                                dict(lmax=1, refine_factor=1), dict(flux=2), dict(flux=1, system=1),
                                dict(flux=1, flux_quad=5), dict(bc=(2, 2, 0, 0, 0, 0), system=1),
                                dict(bc=(2, 2, 0, 0, 0, 0), n0=(2, 16)), dict(bc=(5,) * 6),
                                dict(load_balance=2), dict(load_balance=-1)])
def test_create_rejects_bad_config_before_allocation(kw):
    cfg = _cfg(**kw)
    ptr = C.c_void_p()
    st = ader.lib().ader_create(C.byref(cfg), C.byref(ptr))
    assert st == 2, (kw, st)
    assert not ptr
    assert len(ader.lib().ader_last_error(None)) > 0


def test_struct_layouts_match_the_library():
    L = ader.lib()
    for what, st in enumerate([ader.AderConfig, ader.AderStepReport, ader.AderCell, ader.AderPartitionInfo,
                               ader.AderHaloDesc]):
        assert L.ader_sizeof(what) == C.sizeof(st), st
    assert L.ader_sizeof(99) == -1


def test_abi_version_checked():
    cfg = _cfg()
    cfg.abi_version = 99
    ptr = C.c_void_p()
    assert ader.lib().ader_create(C.byref(cfg), C.byref(ptr)) == 2


@pytest.mark.parametrize("dim,n,ws,bc", [(2, (64, 48), 2, 0), (2, (100, 100), 8, 1), (3, (32, 32, 32), 8, 1),
                                         (3, (256, 256, 256), 4, 1), (3, (20, 30, 40), 6, 0)])
def test_partition_tiles_domain_and_neighbours_are_symmetric(dim, n, ws, bc):
    cfg = _cfg(dim=dim, n0=n, lo=(0,) * dim, hi=(1,) * dim, bc=(bc,) * 6, world_size=ws)
    infos = [ader.ader_partition(cfg, r) for r in range(ws)]
    owner = np.full(n, -1)
    for r, p in enumerate(infos):
        sl = tuple(slice(p.lo[k], p.hi[k]) for k in range(dim))
        assert np.all(owner[sl] == -1)
        owner[sl] = r
        assert p.halo == 3
    assert np.all(owner >= 0)
    for r, p in enumerate(infos):
        for k in range(dim):
            lo_n, hi_n = p.nbr[2 * k], p.nbr[2 * k + 1]
            if lo_n >= 0:
                assert infos[lo_n].nbr[2 * k + 1] == r
            if hi_n >= 0:
                assert infos[hi_n].nbr[2 * k] == r
            if bc == 1:
                assert (lo_n < 0) == (p.lo[k] == 0)
                assert (hi_n < 0) == (p.hi[k] == n[k])


def test_library_is_sm100a_only():
    # the shipped library holds sm_100a SASS (no PTX JIT fallback for other archs)
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ader.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_missing_library_fails_loudly(monkeypatch):
    # the product path has no CPU fallback: without the built extension the
    # binding raises instead of computing anything
    monkeypatch.setattr(ader, "_LIB", None)
    monkeypatch.setattr(ader, "LIB_PATH", os.path.join(ROOT, "no_such_dir", "libader_b200.so"))
    with pytest.raises(ImportError):
        ader.lib()
    with pytest.raises(ImportError):
        ader.Solver(_cfg())
