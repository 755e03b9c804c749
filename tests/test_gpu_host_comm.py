"""Two processes on one GPU whose rank-group collectives go through host
callbacks over a torch.distributed gloo group (ader_create_host_comm): the
per-process path of a multi-GPU run — separate contexts, each issuing its own
halo exchanges, CFL max, error-code max and (AMR) per-level exchanges, index
sums and rebalances in its own order — minus NCCL itself.  Both ranks together
must reproduce one rank bit for bit (the loopback groups of
test_gpu_multirank.py step all ranks in lockstep in one process instead)."""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest

from paper_1212_3585_b200 import ader
from paper_1212_3585_b200 import workloads as W

pytestmark = pytest.mark.gpu

CASES = {
    # periodic in x with 2 ranks: both x neighbours of a rank are the other rank
    "vortex2d_M3_uniform": (dict(dim=2, degree=3, n0=(24, 20), lo=(0, 0), hi=(10, 10), bc=(0,) * 6, cfl=0.9),
                            "vortex", 6),
    "explosion3d_uniform": (dict(dim=3, degree=2, n0=(14, 12, 10), lo=(-1,) * 3, hi=(1,) * 3, bc=(1,) * 6, cfl=0.3),
                            "explosion3", 3),
    "explosion2d_amr_l2": (dict(dim=2, degree=2, n0=(24, 24), lo=(-1, -1), hi=(1, 1), bc=(1,) * 6, lmax=2,
                                cfl=0.45, chi_ref=0.1, chi_rec=0.05, adapt_every=1), "explosion2", 4),
    "explosion2d_amr_l2_balanced": (dict(dim=2, degree=2, n0=(36, 16), lo=(-1, -1), hi=(4, 1), bc=(1,) * 6, lmax=2,
                                         cfl=0.45, chi_ref=0.1, chi_rec=0.05, adapt_every=1, load_balance=1),
                                    "explosion2", 4),
}


def _ic(name):
    return {"vortex": W.isentropic_vortex(), "explosion3": W.explosion(3), "explosion2": W.explosion(2)}[name]


def _rows(cells, nv):
    return sorted((c.level, c.idx[2], c.idx[1], c.idx[0], c.status, tuple(c.u[:nv])) for c in cells)


class GlooComm:
    """ader_host_comm over a gloo process group; per-pair message tags count
    the messages in order, so both sides match them identically."""

    def __init__(self, dist):
        self.dist = dist
        self.sent, self.recd = {}, {}

    def p2p(self, peers, sends, rcounts):
        import torch
        reqs, out = [], [None] * len(peers)
        for i, p in enumerate(peers):
            if len(sends[i]):
                tag = self.sent.get(p, 0)
                self.sent[p] = tag + 1
                reqs.append(self.dist.isend(torch.from_numpy(sends[i]), p, tag=tag))
            if rcounts[i]:
                tag = self.recd.get(p, 0)
                self.recd[p] = tag + 1
                out[i] = torch.empty(rcounts[i], dtype=torch.float64)
                reqs.append(self.dist.irecv(out[i], p, tag=tag))
        for r in reqs:
            r.wait()
        return [o.numpy() if o is not None else None for o in out]

    def allreduce_sum(self, buf):
        import torch
        t = torch.from_numpy(buf.copy())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        buf[:] = t.numpy()

    def allreduce_max_u64(self, buf):
        import torch
        t = torch.from_numpy(buf.view(np.int64).copy())   # speed bits / error codes: < 2^63
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        buf.view(np.int64)[:] = t.numpy()


def _worker(rank, world, port, name, out_dir):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    kw, ic, steps = CASES[name]
    nv = 9 if kw.get("system", 0) == 1 else kw["dim"] + 2
    cfg = ader.make_config(device=0, rank=rank, world_size=world, **kw)
    s = ader.Solver(cfg, comm=GlooComm(dist))
    s.set_initial(_ic(ic))
    rep = s.step(1e300, steps)
    rows = _rows(s.get_cells(), nv)
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump((rows, (rep.dt0, rep.cell_updates, rep.t)), f)
    s.close()
    dist.barrier()
    dist.destroy_process_group()
    assert torch is not None


@pytest.mark.parametrize("name", list(CASES))
def test_two_processes_with_host_collectives_reproduce_one_rank(name):
    import torch.multiprocessing as mp
    kw, ic, steps = CASES[name]
    nv = 9 if kw.get("system", 0) == 1 else kw["dim"] + 2
    one = ader.Solver(ader.make_config(device=0, **{k: v for k, v in kw.items() if k != "load_balance"}))
    one.set_initial(_ic(ic))
    r1 = one.step(1e300, steps)
    ref = _rows(one.get_cells(), nv)
    one.close()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, port, name, d), nprocs=2, join=True, start_method="spawn")
        got = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(2)]
    rows = sorted(sum((g[0] for g in got), []))
    reps = [g[1] for g in got]
    assert all(rp[0] == r1.dt0 for rp in reps)
    assert sum(rp[1] for rp in reps) == r1.cell_updates
    assert len(rows) == len(ref)
    bad = [(a, b) for a, b in zip(rows, ref) if a != b]
    assert not bad, bad[:2]
