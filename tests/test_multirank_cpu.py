"""Multi-rank host logic on CPU (gloo, world_size 2 and 4, no GPU).

The ghost-exchange plan of the CUDA library (ader_partition + ader_halo_plan:
which cells each rank sends, receives, wraps or clamps, and in which axis
order) drives a block-decomposed oracle run over torch.distributed/gloo; the
result must be bitwise identical to the single-domain oracle, because every
cell's arithmetic is local once its ghost cells are exact."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1212_3585_b200 import ader


def smooth_ic(n, dim):
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros((x.shape[0], 9))
        ph = sum(2 * math.pi * (k + 1) * x[:, k] / n[k] for k in range(dim))
        out[:, 0] = 1.0 + 0.2 * np.sin(ph)
        out[:, 1] = 0.3 + 0.1 * np.cos(ph)
        out[:, 2] = -0.2 + 0.1 * np.sin(2 * ph)
        if dim == 3:
            out[:, 3] = 0.1
        out[:, 4] = 1.0 + 0.1 * np.cos(ph)
        return out
    return ic


def explosion_ic(n, dim):
    def ic(x):
        x = np.asarray(x, dtype=np.float64)
        r2 = sum((x[:, k] - n[k] / 2) ** 2 for k in range(dim))
        inside = r2 <= (0.3 * n[0]) ** 2
        out = np.zeros((x.shape[0], 9))
        out[:, 0] = np.where(inside, 1.0, 0.125)
        out[:, 4] = np.where(inside, 1.0, 0.1)
        return out
    return ic


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, ws, port, dim, M, n, bc, icname, steps, q, cfl=0.45):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        cfg = ader.make_config(dim=dim, degree=M, n0=n, lo=(0,) * dim, hi=tuple(float(k) for k in n), bc=bc,
                               world_size=ws, rank=rank, cfl=cfl)
        part = ader.ader_partition(cfg, rank)
        blo = [part.lo[k] for k in range(dim)]
        bhi = [part.hi[k] for k in range(dim)]
        nb = [bhi[k] - blo[k] for k in range(dim)]
        ic = (smooth_ic if icname == "smooth" else explosion_ic)(n, dim)
        # global IC by the oracle, then the rank's block (the oracle's own input)
        g = O.Oracle(dim=dim, degree=M, n=n, lo=(0,) * dim, hi=tuple(float(k) for k in n), bc=bc, cfl=cfl)
        g.set_initial(ic)
        ug = g.get_cells().reshape(tuple(reversed(n)) + (-1,))
        sl = tuple(slice(blo[k], bhi[k]) for k in reversed(range(dim)))
        # the block oracle treats a side shared with another rank as an interior side
        bcb = list(bc) + [0] * (6 - len(bc))
        for a in range(dim):
            for s in (0, 1):
                if ader.ader_halo_plan(cfg, rank, a, s).kind == 1:
                    bcb[2 * a + s] = 0
        o = O.Oracle(dim=dim, degree=M, n=nb, lo=tuple(float(b) for b in blo), hi=tuple(float(b) for b in bhi),
                     bc=bcb, cfl=cfl)
        o.set_cells(ug[sl].reshape(-1, g.nv))
        o.set_external_ghosts(True)
        H = M + 1
        for _ in range(steps):
            u = o.get_padded()                      # (P2, P1, P0, nv)
            if dim == 2:
                u = u.reshape(u.shape[1:])[None]
            for a in range(dim):
                plans = [ader.ader_halo_plan(cfg, rank, a, s) for s in (0, 1)]
                reqs, bufs = [], []

                def box(lo, hi):
                    return (slice(lo[2], hi[2]), slice(lo[1], hi[1]), slice(lo[0], hi[0]))
                for s, p in enumerate(plans):
                    if p.kind == 1:
                        snd = torch.from_numpy(np.ascontiguousarray(u[box(p.send_lo, p.send_hi)]))
                        reqs.append(dist.isend(snd, p.peer, tag=2 * a + s))
                        rcv = torch.zeros(snd.shape, dtype=torch.float64)
                        reqs.append(dist.irecv(rcv, p.peer, tag=2 * a + (1 - s)))
                        bufs.append((p, rcv))
                for r in reqs:
                    r.wait()
                for p, rcv in bufs:
                    u[box(p.recv_lo, p.recv_hi)] = rcv.numpy()
                for s, p in enumerate(plans):
                    if p.kind in (2, 3):
                        lo = list(p.recv_lo)
                        hi = list(p.recv_hi)
                        ax = 2 - a     # numpy axis of grid axis a
                        idx = np.arange(lo[a], hi[a]) - H
                        src = (np.mod(idx, nb[a]) if p.kind == 2 else np.clip(idx, 0, nb[a] - 1)) + H
                        full = list(box(lo, hi))
                        full[ax] = src
                        u[box(lo, hi)] = u[tuple(full[:ax]) + (full[ax],) + tuple(full[ax + 1:])]
            o.set_padded(u.reshape(o.padded_shape()))
            dt = torch.tensor([o.compute_dt()], dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MIN)
            out, _ = o.advance_box(float(dt.item()), [0] * dim, nb)
            o.set_cells(out)
        mine = o.get_cells()
        gathered = [None] * ws
        dist.all_gather_object(gathered, (blo, bhi, mine))
        if rank == 0:
            full = np.zeros(tuple(reversed(n)) + (g.nv,))
            for lo_, hi_, arr in gathered:
                s_ = tuple(slice(lo_[k], hi_[k]) for k in reversed(range(dim)))
                full[s_] = arr.reshape(tuple(hi_[k] - lo_[k] for k in reversed(range(dim))) + (g.nv,))
            g.step(1e300, steps)
            q.put((full.reshape(-1, g.nv), g.get_cells()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws,dim,M,n,bc,icname,cfl", [
    (2, 2, 2, (12, 10), (0,) * 6, "smooth", 0.9),
    (2, 2, 3, (14, 9), (1, 1, 0, 0, 0, 0), "smooth", 0.9),
    (2, 2, 2, (14, 11), (1,) * 6, "explosion", 0.45),
    (4, 3, 2, (8, 8, 6), (1,) * 6, "explosion", 0.3),
])
def test_block_decomposed_run_is_bitwise_identical(ws, dim, M, n, bc, icname, cfl):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, ws, port, dim, M, n, bc, icname, 2, q, cfl)) for r in range(ws)]
    for p in procs:
        p.start()
    full, ref = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(full, ref)
