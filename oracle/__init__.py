"""ctypes loader for the CPU oracle (oracle/ader_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_1212_3585_b200/) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

EULER, MHD = 0, 1
PERIODIC, TRANSMISSIVE, REFLECTIVE, INFLOW, EXACT = 0, 1, 2, 3, 4
RUSANOV, OSHER = 0, 1

IC_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_void_p)


class OrcConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("system", C.c_int32), ("degree", C.c_int32),
        ("n", C.c_int32 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
        ("bc", C.c_int32 * 6),
        ("gamma", C.c_double), ("ch", C.c_double), ("cfl", C.c_double),
        ("pred_tol", C.c_double), ("pred_max_sweeps", C.c_int32),
        ("ic_quad", C.c_int32),
        ("refine_factor", C.c_int32), ("lmax", C.c_int32),
        ("chi_ref", C.c_double), ("chi_rec", C.c_double), ("chi_eps", C.c_double),
        ("flux", C.c_int32), ("flux_quad", C.c_int32),
        ("pred_guess", C.c_int32), ("exact_vel", C.c_double * 3),
    ]


class OrcReport(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("dt", C.c_double),
        ("steps", C.c_int64), ("cell_updates", C.c_int64), ("sweeps_total", C.c_int64),
        ("sweeps_max", C.c_int32), ("updates_per_level", C.c_int64 * 8),
        ("min_threshold_margin", C.c_double),
    ]


def build():
    src = os.path.join(_HERE, "ader_oracle.c")
    so = os.path.join(_HERE, "liboracle.so")
    if (not os.path.exists(so)) or os.path.getmtime(so) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "ader_oracle.h"))):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return so


def lib():
    global _LIB
    if _LIB is None:
        # ORACLE_LIB: a mutated copy of the oracle (tools/oracle_mutation_check.sh
        # shows that the pins fail on it); default: the in-tree build
        _LIB = C.CDLL(os.environ.get("ORACLE_LIB") or build())
        L = _LIB
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(OrcConfig)]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.c_void_p]
        L.orc_set_initial.argtypes = [C.c_void_p, IC_FN, C.c_void_p]
        L.orc_set_initial_box.argtypes = [C.c_void_p, IC_FN, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.orc_set_cells.argtypes = [C.c_void_p, dp]
        L.orc_get_cells.argtypes = [C.c_void_p, dp]
        L.orc_time.restype = C.c_double
        L.orc_time.argtypes = [C.c_void_p]
        L.orc_num_cells.restype = C.c_int64
        L.orc_num_cells.argtypes = [C.c_void_p]
        L.orc_compute_dt.restype = C.c_double
        L.orc_compute_dt.argtypes = [C.c_void_p]
        L.orc_step.argtypes = [C.c_void_p, C.c_double, C.c_int64, C.POINTER(OrcReport)]
        L.orc_advance_box.argtypes = [C.c_void_p, C.c_double, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), dp, C.POINTER(OrcReport)]
        L.orc_dump_recon.argtypes = [C.c_void_p, dp]
        L.orc_dump_pred.argtypes = [C.c_void_p, C.c_double, dp]
        L.orc_dump_flux.argtypes = [C.c_void_p, C.c_double, dp]
        L.orc_nvar.argtypes = [C.c_int, C.c_int]
        L.orc_basis_tables.argtypes = [C.c_int] + [dp] * 5 + [dp, ip, ip, dp] + [dp] * 3
        L.orc_predictor_matrices.argtypes = [C.c_int, C.c_int, dp, dp, dp]
        L.orc_weno_1d.argtypes = [C.c_int, dp, dp]
        L.orc_reconstruct_box.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_predict_cell.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       dp, dp, C.c_double, C.c_int, dp, ip]
        L.orc_face_flux.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_int, C.c_int, C.c_int, dp, dp, dp]
        L.orc_euler_jacobian.argtypes = [C.c_int, C.c_double, dp, C.c_int, dp]
        L.orc_euler_abs_jacobian.argtypes = [C.c_int, C.c_double, dp, C.c_int, dp]
        L.orc_osher.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, dp, dp, C.c_int, dp]
        L.orc_numflux.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, dp, dp,
                                  C.c_int, dp]
        L.orc_phys_flux.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, dp, C.c_int, dp]
        L.orc_max_speed.restype = C.c_double
        L.orc_max_speed.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, dp, C.c_int]
        L.orc_rusanov.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, dp, dp, C.c_int, dp]
        L.orc_prim_to_cons.argtypes = [C.c_int, C.c_int, C.c_double, dp, dp]
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def nvar(system, dim):
    return lib().orc_nvar(system, dim)


def tables(M):
    N = M + 1
    lam, w, p0, p1 = (np.zeros(N) for _ in range(4))
    Sig = np.zeros((N, N))
    rec = np.zeros((4, N, N))
    L = np.zeros(4, dtype=np.int32)
    R = np.zeros(4, dtype=np.int32)
    lin = np.zeros(4)
    M1, Kx1, K1t = (np.zeros((N, N)) for _ in range(3))
    ip = C.POINTER(C.c_int)
    nS = lib().orc_basis_tables(M, _p(lam), _p(w), _p(p0), _p(p1), _p(Sig), _p(rec),
                                L.ctypes.data_as(ip), R.ctypes.data_as(ip), _p(lin),
                                _p(M1), _p(Kx1), _p(K1t))
    return dict(lam=lam, w=w, psi0=p0, psi1=p1, Sigma=Sig, rec=rec[:nS], L=L[:nS], R=R[:nS],
                lin=lin[:nS], M1=M1, Kx1=Kx1, K1t=K1t, nS=nS)


def predictor_matrices(d, M):
    N = M + 1
    NS, NST = N ** d, N ** (d + 1)
    K1 = np.zeros((NST, NST))
    Kd = np.zeros((d, NST, NST))
    F0 = np.zeros((NST, NS))
    lib().orc_predictor_matrices(d, M, _p(K1), _p(Kd), _p(F0))
    return K1, Kd, F0


def weno_1d(M, win):
    win = np.ascontiguousarray(win, dtype=np.float64)
    out = np.zeros(M + 1)
    lib().orc_weno_1d(M, _p(win), _p(out))
    return out


def reconstruct_box(d, M, nv, ubox):
    ubox = np.ascontiguousarray(ubox, dtype=np.float64)
    w = np.zeros((nv, (M + 1) ** d))
    rc = lib().orc_reconstruct_box(d, M, nv, _p(ubox), _p(w))
    assert rc == 0
    return w


def predict_cell(d, M, system, gamma, ch, w, dtdx, tol=1e-13, max_sweeps=32, q0=None):
    w = np.ascontiguousarray(w, dtype=np.float64)
    nv = w.shape[0]
    q = np.zeros((nv, (M + 1) ** (d + 1)))
    dtdx = np.ascontiguousarray(dtdx, dtype=np.float64)
    sw = C.c_int(0)
    L = lib()
    if q0 is None:
        rc = L.orc_predict_cell(d, M, system, gamma, ch, _p(w), _p(dtdx), tol, max_sweeps, _p(q), C.byref(sw))
    else:
        q0 = np.ascontiguousarray(q0, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        L.orc_predict_cell_guess.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, dp, dp, C.c_double,
                                             C.c_int, dp, dp, C.POINTER(C.c_int)]
        rc = L.orc_predict_cell_guess(d, M, system, gamma, ch, _p(w), _p(dtdx), tol, max_sweeps, _p(q0), _p(q),
                                      C.byref(sw))
    return rc, q, sw.value


def extrapolate_guess(d, M, w, qp, r):
    """reading R25: q0 = w + qp(., 1 + r tau) - qp(., 1) at the space-time nodes"""
    w = np.ascontiguousarray(w, dtype=np.float64)
    qp = np.ascontiguousarray(qp, dtype=np.float64)
    q0 = np.zeros_like(qp)
    L = lib()
    dp = C.POINTER(C.c_double)
    L.orc_extrapolate_guess.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, C.c_double, dp]
    L.orc_extrapolate_guess(d, M, w.shape[0], _p(w), _p(qp), r, _p(q0))
    return q0


def face_flux(d, M, system, gamma, ch, direction, qL, qR, flux=RUSANOV, nq=3):
    qL = np.ascontiguousarray(qL, dtype=np.float64)
    qR = np.ascontiguousarray(qR, dtype=np.float64)
    F = np.zeros(qL.shape[0])
    rc = lib().orc_face_flux(d, M, system, gamma, ch, flux, nq, direction, _p(qL), _p(qR), _p(F))
    assert rc == 0
    return F


def phys_flux(system, dim, gamma, ch, u, direction):
    u = np.ascontiguousarray(u, dtype=np.float64)
    f = np.zeros(len(u))
    rc = lib().orc_phys_flux(system, dim, gamma, ch, _p(u), direction, _p(f))
    assert rc == 0
    return f


def max_speed(system, dim, gamma, ch, u, direction):
    u = np.ascontiguousarray(u, dtype=np.float64)
    return lib().orc_max_speed(system, dim, gamma, ch, _p(u), direction)


def rusanov(system, dim, gamma, ch, uL, uR, direction):
    uL = np.ascontiguousarray(uL, dtype=np.float64)
    uR = np.ascontiguousarray(uR, dtype=np.float64)
    f = np.zeros(len(uL))
    rc = lib().orc_rusanov(system, dim, gamma, ch, _p(uL), _p(uR), direction, _p(f))
    assert rc == 0
    return f


def euler_jacobian(dim, gamma, u, direction):
    u = np.ascontiguousarray(u, dtype=np.float64)
    A = np.zeros((len(u), len(u)))
    rc = lib().orc_euler_jacobian(dim, gamma, _p(u), direction, _p(A))
    assert rc == 0
    return A


def euler_abs_jacobian(dim, gamma, u, direction):
    u = np.ascontiguousarray(u, dtype=np.float64)
    A = np.zeros((len(u), len(u)))
    rc = lib().orc_euler_abs_jacobian(dim, gamma, _p(u), direction, _p(A))
    assert rc == 0
    return A


def osher(dim, gamma, uL, uR, direction, nq=3):
    uL = np.ascontiguousarray(uL, dtype=np.float64)
    uR = np.ascontiguousarray(uR, dtype=np.float64)
    f = np.zeros(len(uL))
    rc = lib().orc_osher(EULER, dim, gamma, nq, _p(uL), _p(uR), direction, _p(f))
    assert rc == 0, rc
    return f


def project_subbox(d, M, r, poly, off, tau=0.0, mode=1):
    """Child average of a mother polynomial: mode 1 = q_h(., tau)
    with poly[nv][N^(d+1)], mode 0 = w_h with poly[nv][N^d]."""
    poly = np.ascontiguousarray(poly, dtype=np.float64)
    nv = poly.shape[0]
    out = np.zeros(nv)
    o = (C.c_int * 3)(*((list(off) + [0, 0, 0])[:3]))
    L = lib()
    L.orc_project_subbox.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.c_double, C.POINTER(C.c_double)]
    L.orc_project_subbox(d, M, nv, r, mode, _p(poly), o, tau, _p(out))
    return out


def face_flux_mapped(d, M, system, gamma, ch, direction, qL, offL, sclL, toffL, tsclL,
                     qR, offR, sclR, toffR, tsclR, flux=RUSANOV, nq=3):
    """Space-time face flux over a mapped sub-face x sub-interval (the AMR
    coarse-fine face); None for a side = transmissive boundary."""
    L = lib()
    dp = C.POINTER(C.c_double)
    L.orc_face_flux_mapped.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                       C.c_int, dp, dp, C.c_double, C.c_double, C.c_double,
                                       dp, dp, C.c_double, C.c_double, C.c_double, dp]

    def arr(a):
        return None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    qL, qR = arr(qL), arr(qR)
    oL = np.ascontiguousarray((list(offL) + [0, 0, 0])[:3], dtype=np.float64)
    oR = np.ascontiguousarray((list(offR) + [0, 0, 0])[:3], dtype=np.float64)
    nv = (qL if qL is not None else qR).shape[0]
    F = np.zeros(nv)
    rc = L.orc_face_flux_mapped(d, M, system, gamma, ch, flux, nq, direction,
                                None if qL is None else _p(qL), _p(oL), sclL, toffL, tsclL,
                                None if qR is None else _p(qR), _p(oR), sclR, toffR, tsclR, _p(F))
    assert rc == 0
    return F


def prim_to_cons(system, dim, gamma, prim):
    prim = np.zeros(9) + np.asarray(list(prim) + [0.0] * (9 - len(prim)), dtype=np.float64)
    u = np.zeros(nvar(system, dim))
    lib().orc_prim_to_cons(system, dim, gamma, _p(prim), _p(u))
    return u


class Oracle:
    """Uniform-grid oracle run (level 0 only)."""

    def __init__(self, *, dim, system=EULER, degree, n, lo, hi, bc, gamma=1.4, ch=0.0,
                 cfl=0.9, pred_tol=1e-13, pred_max_sweeps=32, ic_quad=0, flux=RUSANOV, flux_quad=3,
                 pred_guess=0, exact_vel=(0.0, 0.0, 0.0)):
        cfg = OrcConfig()
        cfg.dim, cfg.system, cfg.degree = dim, system, degree
        n = list(n) + [1] * (3 - len(n))
        lo = list(lo) + [0.0] * (3 - len(lo))
        hi = list(hi) + [1.0] * (3 - len(hi))
        for k in range(3):
            cfg.n[k], cfg.lo[k], cfg.hi[k] = n[k], lo[k], hi[k]
        bc = list(bc) + [0] * (6 - len(bc))
        for k in range(6):
            cfg.bc[k] = bc[k]
        cfg.gamma, cfg.ch, cfg.cfl = gamma, ch, cfl
        cfg.pred_tol, cfg.pred_max_sweeps, cfg.ic_quad = pred_tol, pred_max_sweeps, ic_quad
        cfg.flux, cfg.flux_quad = flux, flux_quad
        cfg.pred_guess = pred_guess
        for k in range(3):
            cfg.exact_vel[k] = (list(exact_vel) + [0.0] * 3)[k]
        self.cfg = cfg
        self.dim, self.degree, self.system = dim, degree, system
        self.n = n[:dim]
        self.nv = nvar(system, dim)
        self.ptr = lib().orc_create(C.byref(cfg))
        if not self.ptr:
            raise ValueError("orc_create rejected the configuration")

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().orc_destroy(self.ptr)
            self.ptr = None

    @property
    def ncells(self):
        return int(np.prod(self.n))

    def error(self):
        return lib().orc_last_error(self.ptr).decode()

    def set_initial(self, ic):
        """ic(x[n,3]) -> prim[n,9] (numpy)."""
        def cb(xp, n, pp, user):
            x = np.ctypeslib.as_array(xp, shape=(n, 3))
            p = np.ctypeslib.as_array(pp, shape=(n, 9))
            p[:] = ic(x)
        self._cb = IC_FN(cb)
        rc = lib().orc_set_initial(self.ptr, self._cb, None)
        assert rc == 0

    def set_initial_box(self, ic, blo, bhi):
        def cb(xp, n, pp, user):
            x = np.ctypeslib.as_array(xp, shape=(n, 3))
            p = np.ctypeslib.as_array(pp, shape=(n, 9))
            p[:] = ic(x)
        self._cb = IC_FN(cb)
        a = (C.c_int32 * 3)(*((list(blo) + [0, 0, 0])[:3]))
        b = (C.c_int32 * 3)(*((list(bhi) + [1, 1, 1])[:3]))
        rc = lib().orc_set_initial_box(self.ptr, self._cb, None, a, b)
        assert rc == 0

    def set_cells(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(self.ncells, self.nv)
        lib().orc_set_cells(self.ptr, _p(u))

    def get_cells(self):
        u = np.zeros((self.ncells, self.nv))
        lib().orc_get_cells(self.ptr, _p(u))
        return u

    @property
    def t(self):
        return lib().orc_time(self.ptr)

    def compute_dt(self):
        return lib().orc_compute_dt(self.ptr)

    def step(self, t_end=1e300, max_steps=1):
        rep = OrcReport()
        rc = lib().orc_step(self.ptr, t_end, max_steps, C.byref(rep))
        if rc:
            raise RuntimeError(f"oracle step failed ({rc}): {self.error()}")
        return rep

    def advance_box(self, dt, blo, bhi):
        blo = (list(blo) + [0, 0, 0])[:3]
        bhi = (list(bhi) + [1, 1, 1])[:3]
        a = (C.c_int32 * 3)(*blo)
        b = (C.c_int32 * 3)(*bhi)
        nb = int(np.prod([bhi[k] - blo[k] for k in range(self.dim)]))
        out = np.zeros((nb, self.nv))
        rep = OrcReport()
        rc = lib().orc_advance_box(self.ptr, dt, a, b, _p(out), C.byref(rep))
        if rc:
            raise RuntimeError(f"oracle advance_box failed: {self.error()}")
        return out, rep

    # distributed emulation: padded grid with caller-provided ghost cells
    def padded_shape(self):
        g = self.degree + 1
        p = [k + 2 * g for k in self.n] + ([1] if self.dim == 2 else [])
        return (p[2], p[1], p[0], self.nv)

    def get_padded(self):
        L = lib()
        L.orc_get_padded.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        u = np.zeros(self.padded_shape())
        L.orc_get_padded(self.ptr, _p(u))
        return u

    def set_padded(self, u):
        L = lib()
        L.orc_set_padded.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        u = np.ascontiguousarray(u, dtype=np.float64)
        assert u.shape == self.padded_shape()
        L.orc_set_padded(self.ptr, _p(u))

    def set_external_ghosts(self, on=True):
        L = lib()
        L.orc_set_external_ghosts.argtypes = [C.c_void_p, C.c_int]
        L.orc_set_external_ghosts(self.ptr, 1 if on else 0)

    def dump_recon(self):
        w = np.zeros((self.ncells, self.nv, (self.degree + 1) ** self.dim))
        lib().orc_dump_recon(self.ptr, _p(w))
        return w

    def dump_pred(self, dt):
        q = np.zeros((self.ncells, self.nv, (self.degree + 1) ** (self.dim + 1)))
        rc = lib().orc_dump_pred(self.ptr, dt, _p(q))
        assert rc == 0, self.error()
        return q

    def dump_flux(self, dt):
        e = [k + 1 for k in self.n] + ([1] if self.dim == 2 else [])
        F = np.zeros((self.dim, int(np.prod(e)), self.nv))
        rc = lib().orc_dump_flux(self.ptr, dt, _p(F))
        assert rc == 0, self.error()
        return F


class AmrCell(C.Structure):
    _fields_ = [("level", C.c_int32), ("status", C.c_int32), ("idx", C.c_int64 * 3), ("u", C.c_double * 9)]


def indicator(d, phi, eps=0.01):
    phi = np.ascontiguousarray(phi, dtype=np.float64).reshape(-1)
    L = lib()
    L.orc_indicator.restype = C.c_double
    L.orc_indicator.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_double]
    return L.orc_indicator(d, _p(phi), eps)


class AmrOracle:
    """Cell-by-cell AMR + LTS oracle (oracle/ader_oracle_amr.c)."""

    def __init__(self, *, dim, degree, n, lo, hi, bc, system=EULER, gamma=1.4, ch=0.0, cfl=0.45,
                 refine_factor=3, lmax=1, chi_ref=0.2, chi_rec=0.1, chi_eps=0.01, pred_tol=1e-13,
                 pred_max_sweeps=32, ic_quad=0, flux=RUSANOV, flux_quad=3):
        L = lib()
        vp = C.c_void_p
        L.orc_amr_create.restype = vp
        L.orc_amr_create.argtypes = [C.POINTER(OrcConfig)]
        L.orc_amr_destroy.argtypes = [vp]
        L.orc_amr_last_error.restype = C.c_char_p
        L.orc_amr_last_error.argtypes = [vp]
        L.orc_amr_time.restype = C.c_double
        L.orc_amr_time.argtypes = [vp]
        L.orc_amr_set_initial.argtypes = [vp, IC_FN, vp]
        L.orc_amr_compute_dt.restype = C.c_double
        L.orc_amr_compute_dt.argtypes = [vp]
        L.orc_amr_step.argtypes = [vp, C.c_double, C.c_int64, C.c_int, C.POINTER(OrcReport)]
        L.orc_amr_adapt.argtypes = [vp]
        L.orc_amr_get_cells.restype = C.c_int64
        L.orc_amr_get_cells.argtypes = [vp, C.POINTER(AmrCell)]
        L.orc_amr_check.argtypes = [vp, C.c_char_p, C.c_int]
        L.orc_amr_refine_cell.argtypes = [vp, C.c_int, C.POINTER(C.c_int64)]
        L.orc_amr_schedule.argtypes = [C.POINTER(C.c_int), C.c_int]
        cfg = OrcConfig()
        cfg.dim, cfg.system, cfg.degree = dim, system, degree
        n = list(n) + [1] * (3 - len(n))
        lo = list(lo) + [0.0] * (3 - len(lo))
        hi = list(hi) + [1.0] * (3 - len(hi))
        for k in range(3):
            cfg.n[k], cfg.lo[k], cfg.hi[k] = n[k], lo[k], hi[k]
        bc = list(bc) + [0] * (6 - len(bc))
        for k in range(6):
            cfg.bc[k] = bc[k]
        cfg.gamma, cfg.ch, cfg.cfl = gamma, ch, cfl
        cfg.pred_tol, cfg.pred_max_sweeps, cfg.ic_quad = pred_tol, pred_max_sweeps, ic_quad
        cfg.refine_factor, cfg.lmax = refine_factor, lmax
        cfg.chi_ref, cfg.chi_rec, cfg.chi_eps = chi_ref, chi_rec, chi_eps
        cfg.flux, cfg.flux_quad = flux, flux_quad
        self.cfg, self.dim, self.nv = cfg, dim, nvar(system, dim)
        self.ptr = L.orc_amr_create(C.byref(cfg))
        if not self.ptr:
            raise ValueError("orc_amr_create rejected the configuration")

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().orc_amr_destroy(self.ptr)
            self.ptr = None

    def error(self):
        return lib().orc_amr_last_error(self.ptr).decode()

    def set_initial(self, ic):
        def cb(xp, n, pp, user):
            x = np.ctypeslib.as_array(xp, shape=(n, 3))
            p = np.ctypeslib.as_array(pp, shape=(n, 9))
            p[:] = ic(x)
        self._cb = IC_FN(cb)
        rc = lib().orc_amr_set_initial(self.ptr, self._cb, None)
        if rc:
            raise RuntimeError(self.error())

    @property
    def t(self):
        return lib().orc_amr_time(self.ptr)

    def compute_dt(self):
        return lib().orc_amr_compute_dt(self.ptr)

    def step(self, t_end=1e300, max_steps=1, adapt_every=1):
        rep = OrcReport()
        rc = lib().orc_amr_step(self.ptr, t_end, max_steps, adapt_every, C.byref(rep))
        if rc:
            raise RuntimeError(f"AMR oracle step failed: {self.error()}")
        return rep

    def adapt(self):
        assert lib().orc_amr_adapt(self.ptr) == 0, self.error()

    def margin(self):
        """min threshold margin of the adapts since the last step() / adapt()"""
        L = lib()
        L.orc_amr_margin.restype = C.c_double
        L.orc_amr_margin.argtypes = [C.c_void_p]
        return L.orc_amr_margin(self.ptr)

    def cells(self):
        """structured array: level, status, idx[3], u[9] sorted by (level, z, y, x)"""
        n = lib().orc_amr_get_cells(self.ptr, None)
        arr = (AmrCell * n)()
        lib().orc_amr_get_cells(self.ptr, arr)
        lv = np.array([c.level for c in arr], dtype=np.int32)
        st = np.array([c.status for c in arr], dtype=np.int32)
        ix = np.array([list(c.idx) for c in arr], dtype=np.int64).reshape(-1, 3)
        u = np.array([list(c.u)[:self.nv] for c in arr]).reshape(-1, self.nv)
        return lv, st, ix, u

    def check(self):
        buf = C.create_string_buffer(256)
        rc = lib().orc_amr_check(self.ptr, buf, 256)
        return rc, buf.value.decode()

    def refine_cell(self, level, idx):
        a = (C.c_int64 * 3)(*((list(idx) + [0, 0, 0])[:3]))
        return lib().orc_amr_refine_cell(self.ptr, level, a)

    @staticmethod
    def schedule():
        buf = (C.c_int * 4096)()
        n = lib().orc_amr_schedule(buf, 4096)
        return list(buf[:min(n, 4096)])
