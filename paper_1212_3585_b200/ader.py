"""Thin ctypes binding of the C ABI in include/ader.h (libader_b200.so).

Argument marshalling only: every stage of the path runs in the CUDA kernels
of the library.  There is no fallback: if the shared library is missing or
cannot be loaded, importing the binding's entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libader_b200.so")
_LIB = None

ABI_VERSION = 6
EULER, MHD_GLM = 0, 1
PERIODIC, TRANSMISSIVE, REFLECTIVE, INFLOW = 0, 1, 2, 3
RUSANOV, OSHER = 0, 1
K_WENO, K_PRED, K_FLUX, K_UPDATE, K_HALO, K_OTHER, K_PRED_FLUX, K_COUNT = range(8)
KERNEL_NAMES = ("weno_reconstruct", "stdg_predictor", "face_flux", "fv_update", "halo", "other",
                "stdg_predictor+face_flux")
STATUS = {0: "ADER_OK", 1: "ADER_ERR_ARG", 2: "ADER_ERR_CONFIG", 3: "ADER_ERR_SOLVER", 4: "ADER_ERR_CUDA",
          5: "ADER_ERR_NCCL", 6: "ADER_ERR_UNSUPPORTED"}

IC_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_void_p)


class AderConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("dim", C.c_int32), ("system", C.c_int32), ("degree", C.c_int32),
        ("n0", C.c_int32 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("bc", C.c_int32 * 6),
        ("refine_factor", C.c_int32), ("lmax", C.c_int32),
        ("gamma", C.c_double), ("ch", C.c_double), ("cfl", C.c_double),
        ("chi_ref", C.c_double), ("chi_rec", C.c_double), ("chi_eps", C.c_double),
        ("indicator_var", C.c_int32),
        ("pred_tol", C.c_double), ("pred_max_sweeps", C.c_int32),
        ("ic_quad", C.c_int32), ("adapt_every", C.c_int32),
        ("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
        ("nccl_id", C.c_uint8 * 128),
        ("flux", C.c_int32), ("flux_quad", C.c_int32), ("load_balance", C.c_int32),
        ("pred_guess", C.c_int32), ("exact_vel", C.c_double * 3), ("fuse_pred_flux", C.c_int32),
    ]


class AderStepReport(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("dt0", C.c_double),
        ("macro_steps", C.c_int64), ("cell_updates", C.c_int64), ("updates_per_level", C.c_int64 * 8),
        ("pred_sweeps_total", C.c_int64), ("pred_sweeps_max", C.c_int32), ("rebalances", C.c_int32),
        ("pred_cells", C.c_int64), ("cons_total", C.c_double * 9), ("wall_s", C.c_double),
        ("min_threshold_margin", C.c_double), ("pred_flat_cells", C.c_int64),
    ]


class AderCell(C.Structure):
    _fields_ = [("level", C.c_int32), ("status", C.c_int32), ("idx", C.c_int64 * 3), ("u", C.c_double * 9)]


class AderPartitionInfo(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("coord", C.c_int32 * 3), ("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3),
                ("nbr", C.c_int32 * 6), ("halo", C.c_int32)]


class AderHaloDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("send_lo", C.c_int32 * 3), ("send_hi", C.c_int32 * 3),
                ("recv_lo", C.c_int32 * 3), ("recv_hi", C.c_int32 * 3)]


P2P_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.POINTER(C.c_double)),
                     C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int64))
SUM_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
MAXU_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_uint64), C.c_int64)


class AderHostComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("p2p", P2P_FN), ("allreduce_sum", SUM_FN), ("allreduce_max_u64", MAXU_FN)]


class AderError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libader_b200.so (raises if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.ader_create.argtypes = [C.POINTER(AderConfig), C.POINTER(vp)]
        L.ader_create_host_comm.argtypes = [C.POINTER(AderConfig), C.POINTER(AderHostComm), C.POINTER(vp)]
        L.ader_destroy.argtypes = [vp]
        L.ader_destroy.restype = None
        L.ader_last_error.argtypes = [vp]
        L.ader_last_error.restype = C.c_char_p
        L.ader_set_stream.argtypes = [vp, vp]
        L.ader_set_initial.argtypes = [vp, IC_FN, vp]
        L.ader_set_cells.argtypes = [vp, dp, C.c_int64]
        L.ader_get_state.argtypes = [vp, dp, C.c_int64]
        L.ader_get_cells.argtypes = [vp, C.POINTER(AderCell), C.c_int64, C.POINTER(C.c_int64)]
        L.ader_time.argtypes = [vp]
        L.ader_time.restype = C.c_double
        L.ader_step.argtypes = [vp, C.c_double, C.c_int64, C.POINTER(AderStepReport)]
        L.ader_step_io.argtypes = [vp, dp, dp, C.c_double, C.POINTER(AderStepReport)]
        L.ader_refine.argtypes = [vp, C.POINTER(AderStepReport)]
        L.ader_partition.argtypes = [C.POINTER(AderConfig), C.c_int32, C.POINTER(AderPartitionInfo)]
        L.ader_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.ader_halo_plan.argtypes = [C.POINTER(AderConfig), C.c_int32, C.c_int32, C.c_int32, C.POINTER(AderHaloDesc)]
        L.ader_set_profiling.argtypes = [vp, C.c_int32]
        L.ader_kernel_stats.argtypes = [vp, dp, C.POINTER(C.c_int64), dp]
        L.ader_launch_count.argtypes = [vp, C.POINTER(C.c_int64)]
        L.ader_debug_dump.argtypes = [vp, C.c_int32, C.c_double, dp, C.c_int64]
        L.ader_debug_group_create.argtypes = [C.POINTER(AderConfig), C.c_int32, C.POINTER(vp)]
        L.ader_debug_group_set_initial.argtypes = [C.POINTER(vp), C.c_int32, IC_FN, vp]
        L.ader_debug_group_step.argtypes = [C.POINTER(vp), C.c_int32, C.c_double, C.c_int64,
                                            C.POINTER(AderStepReport)]
        L.ader_sizeof.restype = C.c_int64
        L.ader_sizeof.argtypes = [C.c_int32]
        L.ader_rcb_partition.argtypes = [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int32,
                                         C.POINTER(C.c_int32)]
        _LIB = L
    return _LIB


EXPORTED = ("ader_create", "ader_destroy", "ader_last_error", "ader_set_stream", "ader_set_initial",
            "ader_set_cells", "ader_get_state", "ader_get_cells", "ader_time", "ader_step", "ader_refine",
            "ader_partition", "ader_halo_plan", "ader_nccl_unique_id", "ader_set_profiling", "ader_kernel_stats",
            "ader_launch_count", "ader_debug_dump", "ader_sizeof", "ader_debug_group_create",
            "ader_debug_group_set_initial", "ader_debug_group_step", "ader_rcb_partition",
            "ader_create_host_comm", "ader_step_io")


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_config(*, dim, degree, n0, lo, hi, bc, system=EULER, gamma=1.4, ch=0.0, cfl=0.9,
                refine_factor=3, lmax=0, chi_ref=0.2, chi_rec=0.1, chi_eps=0.01, pred_tol=1e-13,
                pred_max_sweeps=32, ic_quad=0, adapt_every=1, rank=0, world_size=1, device=-1,
                nccl_id=None, flux=RUSANOV, flux_quad=0, load_balance=0, pred_guess=0,
                exact_vel=(0.0, 0.0, 0.0), fuse_pred_flux=None) -> AderConfig:
    cfg = AderConfig()
    cfg.abi_version = ABI_VERSION
    cfg.dim, cfg.system, cfg.degree = dim, system, degree
    n0 = list(n0) + [1] * (3 - len(n0))
    lo = list(lo) + [0.0] * (3 - len(lo))
    hi = list(hi) + [1.0] * (3 - len(hi))
    for k in range(3):
        cfg.n0[k], cfg.lo[k], cfg.hi[k] = n0[k], lo[k], hi[k]
    bc = list(bc) + [0] * (6 - len(bc))
    for k in range(6):
        cfg.bc[k] = bc[k]
    cfg.refine_factor, cfg.lmax = refine_factor, lmax
    cfg.gamma, cfg.ch, cfg.cfl = gamma, ch, cfl
    cfg.chi_ref, cfg.chi_rec, cfg.chi_eps, cfg.indicator_var = chi_ref, chi_rec, chi_eps, 0
    cfg.pred_tol, cfg.pred_max_sweeps = pred_tol, pred_max_sweeps
    cfg.ic_quad, cfg.adapt_every = ic_quad, adapt_every
    cfg.rank, cfg.world_size, cfg.device = rank, world_size, device
    cfg.flux, cfg.flux_quad, cfg.load_balance = flux, flux_quad, load_balance
    cfg.pred_guess = pred_guess
    # uniform grids: 0 = separate predictor and face-flux kernels (default), 1 = the
    # fused tile walk; ADER_FUSE_PRED_FLUX sets the default (A/B tooling)
    if fuse_pred_flux is None:
        fuse_pred_flux = int(os.environ.get("ADER_FUSE_PRED_FLUX", "0"))
    cfg.fuse_pred_flux = fuse_pred_flux
    for k in range(3):
        cfg.exact_vel[k] = (list(exact_vel) + [0.0] * 3)[k]
    if nccl_id is not None:
        for i, b in enumerate(bytes(nccl_id)[:128]):
            cfg.nccl_id[i] = b
    return cfg


def ader_partition(cfg: AderConfig, rank: int) -> AderPartitionInfo:
    info = AderPartitionInfo()
    st = lib().ader_partition(C.byref(cfg), rank, C.byref(info))
    if st:
        raise AderError(st, "ader_partition rejected the configuration")
    return info


def ader_rcb_partition(dim: int, n0, weights, world: int):
    """Level-0 blocks of the dynamic load balancing (ader.h: ader_rcb_partition):
    weights[z][y][x] (x fastest in memory) -> [(lo[3], hi[3])] per rank."""
    import numpy as np
    n = list(n0) + [1] * (3 - len(n0))
    w = np.ascontiguousarray(weights, dtype=np.int64).reshape(-1)
    if w.size != n[0] * n[1] * n[2]:
        raise ValueError("weights must have n0[0]*n0[1]*n0[2] entries")
    boxes = (C.c_int32 * (6 * world))()
    st = lib().ader_rcb_partition(dim, (C.c_int32 * 3)(*n), w.ctypes.data_as(C.POINTER(C.c_int64)), world, boxes)
    if st:
        raise AderError(st, "ader_rcb_partition rejected the arguments")
    return [(tuple(boxes[6 * p:6 * p + 3]), tuple(boxes[6 * p + 3:6 * p + 6])) for p in range(world)]


def ader_halo_plan(cfg: AderConfig, rank: int, axis: int, side: int) -> AderHaloDesc:
    d = AderHaloDesc()
    st = lib().ader_halo_plan(C.byref(cfg), rank, axis, side, C.byref(d))
    if st:
        raise AderError(st, "ader_halo_plan rejected the arguments")
    return d


def ader_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = lib().ader_nccl_unique_id(buf)
    if st:
        raise AderError(st, "ncclGetUniqueId failed")
    return bytes(buf)


def host_comm(obj) -> AderHostComm:
    """ader_host_comm over a Python object with methods
        p2p(peers, sends, recv_counts) -> list of received numpy arrays
        allreduce_sum(np.ndarray) -> None (in place)
        allreduce_max_u64(np.ndarray) -> None (in place)
    (e.g. a torch.distributed gloo group).  Marshalling only."""
    def p2p(user, n, peers, send, scount, recv, rcount):
        try:
            pe = [peers[i] for i in range(n)]
            sends = [np.ctypeslib.as_array(send[i], shape=(scount[i],)).copy() if scount[i] else
                     np.zeros(0) for i in range(n)]
            got = obj.p2p(pe, sends, [rcount[i] for i in range(n)])
            for i in range(n):
                if rcount[i]:
                    np.ctypeslib.as_array(recv[i], shape=(rcount[i],))[:] = got[i]
            return 0
        except Exception as e:   # noqa: BLE001 — reported to the library as a failed collective
            print("ader host p2p failed:", e)
            return 1

    def asum(user, buf, n):
        try:
            obj.allreduce_sum(np.ctypeslib.as_array(buf, shape=(n,)))
            return 0
        except Exception as e:   # noqa: BLE001
            print("ader host allreduce_sum failed:", e)
            return 1

    def amax(user, buf, n):
        try:
            obj.allreduce_max_u64(np.ctypeslib.as_array(buf, shape=(n,)))
            return 0
        except Exception as e:   # noqa: BLE001
            print("ader host allreduce_max failed:", e)
            return 1

    hc = AderHostComm()
    hc.p2p, hc.allreduce_sum, hc.allreduce_max_u64 = P2P_FN(p2p), SUM_FN(asum), MAXU_FN(amax)
    hc._keep = (hc.p2p, hc.allreduce_sum, hc.allreduce_max_u64, obj)
    return hc


class Solver:
    """One rank's context: ader_create ... ader_destroy (comm: optional host
    collectives, ader_create_host_comm)."""

    def __init__(self, cfg: AderConfig, comm=None):
        self.cfg = cfg
        self.nv = 9 if cfg.system == MHD_GLM else cfg.dim + 2
        self.N = cfg.degree + 1
        self.part = ader_partition(cfg, cfg.rank)
        self.block = [self.part.hi[k] - self.part.lo[k] for k in range(cfg.dim)]
        self.ptr = C.c_void_p()
        self._comm = host_comm(comm) if comm is not None else None
        if self._comm is not None:
            st = lib().ader_create_host_comm(C.byref(cfg), C.byref(self._comm), C.byref(self.ptr))
        else:
            st = lib().ader_create(C.byref(cfg), C.byref(self.ptr))
        if st:
            raise AderError(st, lib().ader_last_error(None).decode())

    def close(self):
        if self.ptr:
            lib().ader_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        if st:
            raise AderError(st, lib().ader_last_error(self.ptr).decode())

    @property
    def ncells(self):
        return int(np.prod(self.block))

    def set_stream(self, stream_ptr):
        self._chk(lib().ader_set_stream(self.ptr, C.c_void_p(stream_ptr)))

    def set_initial(self, ic):
        def cb(xp, n, pp, user):
            x = np.ctypeslib.as_array(xp, shape=(n, 3))
            p = np.ctypeslib.as_array(pp, shape=(n, 9))
            p[:] = ic(x)
        self._cb = IC_FN(cb)
        self._chk(lib().ader_set_initial(self.ptr, self._cb, None))

    def set_cells(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        self._chk(lib().ader_set_cells(self.ptr, _dp(u), self.ncells))

    def set_cells_ptr(self, host_ptr):
        self._chk(lib().ader_set_cells(self.ptr, C.cast(C.c_void_p(host_ptr), C.POINTER(C.c_double)), self.ncells))

    def get_state(self, out=None):
        if out is None:
            out = np.empty((self.ncells, self.nv))
        self._chk(lib().ader_get_state(self.ptr, _dp(out), self.ncells))
        return out

    def get_state_ptr(self, host_ptr):
        self._chk(lib().ader_get_state(self.ptr, C.cast(C.c_void_p(host_ptr), C.POINTER(C.c_double)), self.ncells))

    def get_cells(self):
        n = C.c_int64(0)
        self._chk(lib().ader_get_cells(self.ptr, None, 0, C.byref(n)))
        arr = (AderCell * n.value)()
        self._chk(lib().ader_get_cells(self.ptr, arr, n.value, C.byref(n)))
        return arr

    @property
    def t(self):
        return lib().ader_time(self.ptr)

    def step(self, t_end=1e300, max_steps=1) -> AderStepReport:
        rep = AderStepReport()
        self._chk(lib().ader_step(self.ptr, t_end, max_steps, C.byref(rep)))
        return rep

    def step_io(self, host_in, host_out, t_end=1e300) -> AderStepReport:
        """One macro step with the state crossing the host boundary (ader_step_io):
        host_in / host_out are numpy arrays or raw pointers (int) of
        [owned cell][nu] doubles; host_in may be None."""
        def ptr(a):
            if a is None:
                return None
            if isinstance(a, int):
                return C.cast(C.c_void_p(a), C.POINTER(C.c_double))
            return _dp(a)
        rep = AderStepReport()
        self._chk(lib().ader_step_io(self.ptr, ptr(host_in), ptr(host_out), t_end, C.byref(rep)))
        return rep

    def refine(self):
        rep = AderStepReport()
        self._chk(lib().ader_refine(self.ptr, C.byref(rep)))
        return rep

    def set_profiling(self, on):
        self._chk(lib().ader_set_profiling(self.ptr, 1 if on else 0))

    def kernel_stats(self):
        ms = np.zeros(K_COUNT)
        ln = np.zeros(K_COUNT, dtype=np.int64)
        fl = np.zeros(K_COUNT)
        self._chk(lib().ader_kernel_stats(self.ptr, _dp(ms), ln.ctypes.data_as(C.POINTER(C.c_int64)), _dp(fl)))
        return ms, ln, fl

    def launch_count(self):
        n = C.c_int64(0)
        self._chk(lib().ader_launch_count(self.ptr, C.byref(n)))
        return n.value

    def debug_dump(self, what, dt=0.0):
        d, nv, N = self.cfg.dim, self.nv, self.N
        nc = self.ncells
        if what == 0:
            out = np.zeros((nc, nv, N ** d))
        elif what == 1:
            out = np.zeros((nc, nv, N ** (d + 1)))
        else:
            e = [b + 1 for b in self.block] + ([1] if d == 2 else [])
            out = np.zeros((d, int(np.prod(e)), nv))
        self._chk(lib().ader_debug_dump(self.ptr, what, dt, _dp(out), out.size))
        return out


class LoopbackGroup:
    """Test-only: the n ranks of a partition as contexts in this process on one
    GPU, stepped in lockstep with device-copy halo exchange (ader_debug_group_*)."""

    def __init__(self, cfg: AderConfig, n: int):
        self.cfg, self.n = cfg, n
        self.ptrs = (C.c_void_p * n)()
        st = lib().ader_debug_group_create(C.byref(cfg), n, self.ptrs)
        if st:
            raise AderError(st, lib().ader_last_error(None).decode())
        self.nv = 9 if cfg.system == MHD_GLM else cfg.dim + 2
        self.parts = []
        for r in range(n):
            c = AderConfig.from_buffer_copy(cfg)
            c.rank, c.world_size = r, n
            self.parts.append(ader_partition(c, r))

    def close(self):
        for i in range(self.n):
            if self.ptrs[i]:
                lib().ader_destroy(self.ptrs[i])
                self.ptrs[i] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_initial(self, ic):
        def cb(xp, n, pp, user):
            x = np.ctypeslib.as_array(xp, shape=(n, 3))
            p = np.ctypeslib.as_array(pp, shape=(n, 9))
            p[:] = ic(x)
        self._cb = IC_FN(cb)
        st = lib().ader_debug_group_set_initial(self.ptrs, self.n, self._cb, None)
        if st:
            raise AderError(st, lib().ader_last_error(self.ptrs[0]).decode())

    def step(self, t_end=1e300, max_steps=1):
        reps = (AderStepReport * self.n)()
        st = lib().ader_debug_group_step(self.ptrs, self.n, t_end, max_steps, reps)
        if st:
            raise AderError(st, lib().ader_last_error(self.ptrs[0]).decode())
        return list(reps)

    def get_cells(self):
        """AMR: the union of the ranks' own subtrees, as ader_cell records."""
        out = []
        for i in range(self.n):
            n = C.c_int64(0)
            st = lib().ader_get_cells(self.ptrs[i], None, 0, C.byref(n))
            arr = (AderCell * n.value)()
            if not st:
                st = lib().ader_get_cells(self.ptrs[i], arr, n.value, C.byref(n))
            if st:
                raise AderError(st, lib().ader_last_error(self.ptrs[i]).decode())
            out.extend(arr)
        return out

    def gather(self):
        """Global state [z][y][x][nv] assembled from the ranks' owned blocks."""
        d = self.cfg.dim
        n0 = [self.cfg.n0[k] for k in range(3)]
        out = np.zeros((n0[2], n0[1], n0[0], self.nv))
        for i, pi in enumerate(self.parts):
            lo = [pi.lo[k] for k in range(3)]
            hi = [pi.hi[k] for k in range(3)]
            if d == 2:
                lo[2], hi[2] = 0, 1
            cnt = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2])
            buf = np.empty((cnt, self.nv))
            st = lib().ader_get_state(self.ptrs[i], _dp(buf), cnt)
            if st:
                raise AderError(st, lib().ader_last_error(self.ptrs[i]).decode())
            out[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = buf.reshape(hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0],
                                                                     self.nv)
        return out
