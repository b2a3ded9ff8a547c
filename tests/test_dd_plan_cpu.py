"""Domain-decomposition halo maps on CPU, no GPU:
relcp_dd_plan_host is host code inside librelcp.so.

* every part's plan is consistent with every other part's (what p sends to q
  is what q expects from p, body for body, in the same order);
* world_size-2 gloo processes (one part each) run the DD wrench with those
  maps: each rank sums its own rows' wrench terms over its local bodies
  (owned + ghosts), ships the ghost partials to their owners over gloo, and
  the owners add them in ascending part order; the result on every owned body
  equals the oracle's single-domain F = D x to 1e-12.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import scenes


def _net(seed=3, n=600, m=2400, local=True):
    if local:
        b, ia, ib, nrm, ra, rb = scenes.local_constraint_network(n, m, seed)
    else:
        b, ia, ib, nrm, ra, rb = scenes.random_constraint_network(n, m, seed)
    return b, ia, ib, nrm, np.cross(ra, nrm), np.cross(rb, nrm)


def _offsets(n, K, empty=None):
    off = [round(k * n / K) for k in range(K + 1)]
    if empty is not None:  # make part `empty` own nothing
        off[empty + 1] = off[empty]
    return np.array(off, dtype=np.int64)


@pytest.mark.parametrize("K,local,empty", [(2, True, None), (3, False, None), (5, True, 2), (4, False, 0)])
def test_dd_plans_agree(K, local, empty):
    from paper_2506_14097_b200 import relcp as R
    b, ia, ib, *_ = _net(local=local)
    off = _offsets(b["n"], K, empty)
    plans = [R.dd_plan_host(off, ia, ib, k) for k in range(K)]
    n_rows = 0
    for k, P in enumerate(plans):
        inf = P["info"]
        lo, hi = off[k], off[k + 1]
        assert inf["n_own"] == hi - lo
        rows = np.arange(inf["row_lo"], inf["row_hi"])
        assert np.all((ia[rows] >= lo) & (ia[rows] < hi))
        n_rows += len(rows)
        outside = ib[rows][(ib[rows] < lo) | (ib[rows] >= hi)]
        assert np.array_equal(P["ghost"], np.unique(outside))
        for q in range(K):  # ghost segment q = the ghosts owned by q
            seg = P["ghost"][P["gseg"][q]:P["gseg"][q + 1]]
            assert np.all((seg >= off[q]) & (seg < off[q + 1]))
    assert n_rows == len(ia)
    for q, Pq in enumerate(plans):
        for p, Pp in enumerate(plans):
            if p == q:
                assert Pq["rseg"][p + 1] == Pq["rseg"][p]
                continue
            sent = Pp["ghost"][Pp["gseg"][q]:Pp["gseg"][q + 1]]
            got = Pq["recv_list"][Pq["rseg"][p]:Pq["rseg"][p + 1]]
            assert np.array_equal(got, sent - off[q])


def test_dd_plan_rejects_unsorted():
    from paper_2506_14097_b200 import relcp as R
    b, ia, ib, *_ = _net()
    with pytest.raises(R.RelcpError):
        R.dd_plan_host(_offsets(b["n"], 2), ia[::-1].copy(), ib[::-1].copy(), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_wrench(rows, ia_l, ib_l, nrm, ta, tb, x, n_loc):
    """Plain per-row accumulation of -[n; t_a] x on a, +[n; t_b] x on b."""
    F = np.zeros((n_loc, 6))
    for r, a, bb in zip(rows, ia_l, ib_l):
        F[a, :3] -= nrm[r] * x[r]
        F[a, 3:] -= ta[r] * x[r]
        F[bb, :3] += nrm[r] * x[r]
        F[bb, 3:] += tb[r] * x[r]
    return F


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_14097_b200 import relcp as R
    b, ia, ib, nrm, ta, tb = _net(seed=9, n=500, m=2000)
    x = np.random.default_rng(4).standard_normal(len(ia))
    off = _offsets(b["n"], world)
    P = R.dd_plan_host(off, ia, ib, rank)
    inf = P["info"]
    lo, hi, n_own = off[rank], off[rank + 1], inf["n_own"]
    rows = np.arange(inf["row_lo"], inf["row_hi"])
    ghost = P["ghost"]
    ib_l = np.where((ib[rows] >= lo) & (ib[rows] < hi), ib[rows] - lo, n_own + np.searchsorted(ghost, ib[rows]))
    F = _local_wrench(rows, ia[rows] - lo, ib_l, nrm, ta, tb, x, n_own + len(ghost))
    # ghost partials -> owners (variable-size blocks, flat float64)
    send = [torch.from_numpy(F[n_own + P["gseg"][q]:n_own + P["gseg"][q + 1]].ravel().copy()) for q in range(world)]
    recv = [torch.empty(6 * int(P["rseg"][p + 1] - P["rseg"][p]), dtype=torch.float64) for p in range(world)]
    reqs = []
    for q in range(world):  # gloo has no all_to_all: point-to-point per peer
        if q != rank and send[q].numel():
            reqs.append(dist.isend(send[q], q))
        if q != rank and recv[q].numel():
            reqs.append(dist.irecv(recv[q], q))
    for r in reqs:
        r.wait()
    Fo = F[:n_own].copy()
    for p in range(world):  # ascending source part: the library's fixed order
        if p == rank:
            continue
        slots = P["recv_list"][P["rseg"][p]:P["rseg"][p + 1]]
        blk = recv[p].numpy().reshape(-1, 6)
        for j, v in zip(slots, blk):
            Fo[j] += v
    out[rank] = (int(lo), Fo)
    dist.destroy_process_group()


def test_dd_wrench_exchange_gloo_world2(orc):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    b, ia, ib, nrm, ta, tb = _net(seed=9, n=500, m=2000)
    x = np.random.default_rng(4).standard_normal(len(ia))
    W = orc.body_W(b)
    F_ref, _ = orc.wrench(W, ia, ib, nrm, ta, tb, x)
    F = np.zeros_like(F_ref)
    for r in range(2):
        lo, Fo = out[r]
        F[lo:lo + len(Fo)] = Fo
    assert np.max(np.abs(F - F_ref)) <= 1e-12 * np.max(np.abs(F_ref))
