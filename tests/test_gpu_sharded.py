"""Subdomain-sharded solve (dgas_shard_* + dgas.ShardedSolver) on the GPU.

The single-GPU box has one device, so the ranks here are processes on cuda:0 with gloo collectives
(host-mediated: no rank's kernel ever waits on another rank's kernel). Each rank runs only its own
subdomains / rows / cells through the dgas_shard_* kernels; the result must match the oracle's PCG
(north_star tolerances) and the single-GPU dgas_pcg on the same problem."""
import os
import socket

import numpy as np
import pytest

import dgas_gen as g
import oracle as O

pytestmark = pytest.mark.gpu

CASES = {
    "cfg1": lambda: g.config(1),
    "cfg2": lambda: g.config(2),
    "cfg4s": lambda: g.config(4, scale="small"),
    "cfg3s": lambda: g.config(3, scale="small"),
    "ex4_h256_H16_p3": lambda: g.paper_case(4, 256, 16, 3),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(name, rank, world):
    """One rank: the sharded solve, the oracle's PCG on the same b, and (when the stopping iterations
    differ, R22) both again at the common iteration count."""
    import torch
    from paper_1903_11357_b200 import dgas
    torch.cuda.set_device(0)
    P = CASES[name]()
    S = dgas.Solver(P)
    o = O.Oracle(P)
    o.setup_schwarz()
    b = o.rhs()
    bt = torch.from_numpy(b).cuda()
    SS = dgas.ShardedSolver(S)
    x, it, cond, st = SS.pcg(bt, rtol=1e-8)
    ref = o.pcg(b, rtol=1e-8)
    res = dict(it=it, cond=cond, st=st, ref_it=ref["iters"], ref_cond=ref["cond"], x=x.cpu().numpy(),
               own=(SS.B.dof_begin, SS.B.dof_end), N=S.N)
    if it == ref["iters"]:
        res["xerr"] = float(np.linalg.norm(res["x"] - ref["x"]) / np.linalg.norm(ref["x"]))
    else:
        k = min(it, ref["iters"])
        xk, ik, _, _ = SS.pcg(bt, rtol=1e-300, maxit=k)
        rk = o.pcg(b, rtol=1e-300, maxit=k)
        res["xerr"] = float(np.linalg.norm(xk.cpu().numpy() - rk["x"]) / np.linalg.norm(rk["x"]))
    S.close()
    return res


def _check(name, res):
    """north_star tolerances against the oracle: iterations (+-2, else the oracle's own rounding spread,
    parity_helpers._iters_ok), x 1e-7 (at the common iteration count), K 1%."""
    from parity_helpers import _iters_ok
    assert res["st"] == 0
    if abs(res["it"] - res["ref_it"]) > 2:
        P = CASES[name]()
        o = O.Oracle(P)
        o.setup_schwarz()
        b = o.rhs()
        assert _iters_ok(o, b, o.pcg(b, rtol=1e-8), res["it"], P, f"sharded {name}"), (res["it"], res["ref_it"])
    assert res["xerr"] <= 1e-7, res["xerr"]
    assert abs(res["cond"] - res["ref_cond"]) <= 0.01 * res["ref_cond"], (res["cond"], res["ref_cond"])


@pytest.mark.parametrize("name", ["cfg1", "cfg4s"])
def test_sharded_single_rank(name):
    """World size 1 (no process group): the sharded kernels over the whole range."""
    res = _run(name, 0, 1)
    _check(name, res)


def _worker(rank, world, port, name, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = _run(name, rank, world)
    except Exception as e:  # report in the parent
        out[rank] = {"error": repr(e)}
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg4s", 2), ("cfg3s", 3), ("ex4_h256_H16_p3", 2)])
def test_sharded_multi_rank(name, world):
    import torch.multiprocessing as mp
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, name, out), nprocs=world, join=True)
    ranges = []
    for r in range(world):
        assert "error" not in out[r], out[r]
        _check(name, out[r])
        ranges.append(out[r]["own"])
        # every rank ends with the same full solution (x summed over the ranks' own dofs)
        assert np.array_equal(out[r]["x"], out[0]["x"])
    # the ranks' own ranges tile the dofs
    ranges.sort()
    assert ranges[0][0] == 0 and all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    assert ranges[-1][1] == out[0]["N"]
