"""Multi-rank paths on CPU (gloo): bench.py's max-over-ranks timing / summed work, and the collective
schedule of the subdomain-sharded solver (dgas.ShardedSolver) with an oracle-backed mock
of its per-rank kernels (the kernels themselves are checked against the single-GPU solve in -m gpu)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, iters = bench.aggregate(10.0 + 5 * rank, 100 + rank, world, device="cpu")
    out[rank] = (ms, iters)
    dist.barrier()
    dist.destroy_process_group()


def test_aggregate_world2_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        ms, iters = out[r]
        assert ms == 15.0          # max over ranks
        assert iters == 201.0      # work of all replicas


def test_aggregate_single_rank():
    import bench
    assert bench.aggregate(3.0, 7, 1) == (3.0, 7)


# --------------------------------------------------------------------------- sharded solve (NEXT-3)
class OracleShardMock:
    """CPU stand-in for dgas.ShardBackend (tests only): the dgas_shard_* buffer semantics of
    include/dgas.h, computed from the ORACLE's dense operators on this rank's subdomains. Checks the
    ShardedSolver driver's collective schedule, not the kernels (those run in the -m gpu test)."""

    def __init__(self, P, o, A, Q, A0, rank, nranks):
        import numpy as np
        import torch
        self.np_, self.torch = np, torch
        subs = np.array_split(np.arange(P.n_sub), nranks)[rank]
        self.own_cells = np.isin(P.part, subs)
        self.own = np.repeat(self.own_cells, P.n_p)
        self.o, self.A, self.Q, self.A0 = o, A, Q, A0
        self.N, self.N0, self.cap = o.N, o.N0, o.N  # halo buffer = p on own dofs, zero elsewhere
        self.s = {}

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64)

    def _set(self, t, v):
        t.copy_(self.torch.from_numpy(self.np_.ascontiguousarray(v, dtype=self.np_.float64)))

    def begin(self, b, red0):
        np = self.np_
        self.b = b.numpy().copy()
        self.x = np.zeros(self.N); self.r = self.b.copy(); self.p = np.zeros(self.N)
        self.alphas, self.betas, self.rz = [], [], 0.0
        ro = np.where(self.own, self.r, 0)
        self._set(red0, np.concatenate([self.Q.T @ ro, [ro @ ro, (self.b * self.own) @ self.b]]))

    def precond(self, red0, red1):
        np = self.np_
        z0 = np.linalg.solve(self.A0, red0.numpy()[:self.N0])
        ro = np.where(self.own, self.r, 0)
        zl = self.o_local.apply(ro)  # local solves: zero outside the own subdomains since ro is
        self.z = np.where(self.own, zl + self.Q @ z0, 0)
        self._set(red1, [ro @ self.z])

    def direction(self, red1, hsend, first):
        rz = float(red1[0])
        if first:
            self.p = self.z.copy()
        else:
            beta = rz / self.rz
            self.betas.append(beta)
            self.p = self.np_.where(self.own, self.z + beta * self.p, 0)
        self.rz = rz
        self._set(hsend, self.np_.where(self.own, self.p, 0))

    def spmv(self, hall, red2):
        pfull = hall.numpy().reshape(-1, self.N).sum(0)  # every rank's own p
        self.p = pfull
        self.q = self.A @ pfull
        self._set(red2, [(self.np_.where(self.own, pfull, 0)) @ self.q])

    def update(self, red2, red0):
        np = self.np_
        alpha = self.rz / float(red2[0])
        self.alphas.append(alpha)
        self.x = np.where(self.own, self.x + alpha * self.p, 0)
        self.r = np.where(self.own, self.r - alpha * self.q, 0)
        self._set(red0, np.concatenate([self.Q.T @ self.r, [self.r @ self.r, 0.0]]))

    def finish(self, iters, x, lz):
        import oracle as O
        self._set(x, self.np_.where(self.own, self.x, 0))
        if iters:
            self._set(lz, O.lanczos(self.alphas[:iters], self.betas[:max(iters - 1, 0)]))
        return 0


def _shard_worker(rank, world, port, out):
    import numpy as np
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import dgas_gen as g
    import oracle as O
    import torch
    from paper_1903_11357_b200 import dgas
    P = g.config(2, scale="small")
    o = O.Oracle(P)
    o.setup_schwarz()
    A = o.dense_A()
    f, c, _, _ = o._ov
    Q = np.zeros((o.N, o.N0))
    G = o.G()
    for k in range(o.n_ov):
        Q[f[k] * o.np_:(f[k] + 1) * o.np_, c[k] * o.nq_:(c[k] + 1) * o.nq_] += G[k]
    mock = OracleShardMock(P, o, A, Q, o.A0(), rank, world)
    mock.o_local = O.Oracle(P)
    mock.o_local.setup_schwarz(use_coarse=False)
    S = dgas.ShardedSolver(backend=mock)
    b = o.rhs()
    x, it, cond, st = S.pcg(torch.from_numpy(b), rtol=1e-8)
    ref = o.pcg(b, rtol=1e-8)
    out[rank] = (it, ref["iters"], float(np.linalg.norm(x.numpy() - ref["x"]) / np.linalg.norm(ref["x"])),
                 cond, ref["cond"], st)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_driver_schedule_gloo(world):
    """ShardedSolver's collective schedule (sum of [Q^T r | r.r | b.b], r.z, p.q; all-gather of the halo)
    on world_size 2 and 3 gloo ranks, each owning a block of subdomains, reproduces the single-process
    oracle PCG: same iteration count, x to 1e-10, Lanczos K to 1e-5."""
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        it, it_ref, relx, cond, cond_ref, st = out[r]
        assert st == 0 and it == it_ref, (it, it_ref)
        assert relx <= 1e-10, relx
        assert abs(cond - cond_ref) <= 1e-5 * cond_ref  # Ritz value: rounding of the sums moves it ~1e-6
