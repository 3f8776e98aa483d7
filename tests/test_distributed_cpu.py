"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The node-partitioned condensing (paper_2602_17601_b200/partition.py) is run
with the real partition plan, the real point-to-point halo exchange and the
real all-reduce; the per-rank stage update is a NumPy restatement of K-REC
restricted to owned nodes.  Gamma rows and the all-reduced H/g must equal the
single-process oracle (condensing.py:182-228, :363-406).
"""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref_port as O
from paper_2602_17601_b200.batch import shard_range
from paper_2602_17601_b200.graph import chain_topology, mesh_topology
from paper_2602_17601_b200.partition import (allreduce_sum, exchange_rows, gather_owned,
                                             partition_nodes)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance(topo, N=4, nx=2, nu=1, seed=3):
    rng = np.random.default_rng(seed)
    M, E = topo.node_count, len(topo.edges)
    lin = SimpleNamespace(topology=topo, horizon=N,
                          a_self=rng.standard_normal((N, M, nx, nx)) * 0.4,
                          a_nbr=rng.standard_normal((N, E, nx, nx)) * 0.3,
                          b=rng.standard_normal((N, M, nx, nu)), c=rng.standard_normal((N, M, nx)),
                          n_state=nx, n_u=nu)
    q = rng.standard_normal((M, N + 1, nx, nx))
    q = np.einsum("mkab,mkcb->mkac", q, q) * 0.3
    spec = SimpleNamespace(topology=topo, horizon=N, q=q, x_ref=rng.standard_normal((M, N + 1, nx)),
                           r=np.tile(np.eye(nu), (N, 1, 1)), u_ref=np.zeros((N, nu)),
                           input_constraints=None, state_constraints=[])
    return lin, spec, rng.standard_normal((M, nx))


def _worker(rank, world, port, graph, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        topo = chain_topology(11) if graph == "chain" else mesh_topology(5, 4)
        lin, spec, x0 = _instance(topo)
        N, nx, nu = lin.horizon, lin.n_state, lin.n_u
        M = topo.node_count
        part = partition_nodes(topo, world, rank)
        ptr, src = topo.csr()
        W = torch.zeros((M, N + 1, nx, 1 + N * nu), dtype=torch.float64)
        W[part.lo:part.hi, 0, :, 0] = torch.from_numpy(x0[part.lo:part.hi])
        exchange_rows(part, W, stage_slice=0)
        for n in range(N):
            live = 1 + n * nu
            prev = W[:, n].numpy()
            for i in range(part.lo, part.hi):
                acc = lin.a_self[n, i] @ prev[i, :, :live]
                for e in range(ptr[i], ptr[i + 1]):
                    acc = acc + lin.a_nbr[n, e] @ prev[src[e], :, :live]
                acc[:, 0] += lin.c[n, i]
                W[i, n + 1, :, :live] = torch.from_numpy(acc)
                W[i, n + 1, :, live:live + nu] = torch.from_numpy(lin.b[n, i])
            exchange_rows(part, W, stage_slice=n + 1)
        Wn = W.numpy()
        gu, gx = Wn[..., 1:], Wn[..., 0]
        # partial cost over owned nodes, R-bar on rank 0 only, then all-reduce
        q_lin = -2.0 * np.einsum("mkab,mkb->mka", spec.q, spec.x_ref)
        H = np.zeros((N * nu, N * nu))
        g = np.zeros(N * nu)
        if rank == 0:
            H, gr = O.r_bar(spec)
            g = gr.copy()
        for k in range(1, N + 1):
            sl = slice(part.lo, part.hi)
            Gk = gu[sl, k, :, : k * nu]
            H[: k * nu, : k * nu] += np.tensordot(Gk, spec.q[sl, k] @ Gk, axes=([0, 1], [0, 1]))
            wk = 2.0 * (spec.q[sl, k] @ gx[sl, k, :, None])[..., 0] + q_lin[sl, k]
            g[: k * nu] += np.einsum("mab,ma->b", Gk, wk)
        Ht, gt = torch.from_numpy(H), torch.from_numpy(g)
        allreduce_sum(Ht)
        allreduce_sum(gt)
        gather_owned(part, W)
        out[rank] = (W.numpy().copy(), Ht.numpy().copy(), gt.numpy().copy(),
                     {p: v.tolist() for p, v in part.halo.items()},
                     {p: v.tolist() for p, v in part.send.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("graph,world", [("chain", 2), ("mesh", 2), ("mesh", 3)])
def test_partitioned_condensing_matches_single_process(graph, world):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, graph, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    topo = chain_topology(11) if graph == "chain" else mesh_topology(5, 4)
    lin, spec, x0 = _instance(topo)
    gu, gx = O.condense_gammas(lin, x0)
    qp = O.condense_ocp(spec, lin, x0, gammas=(gu, gx))
    H_ref = qp.h  # symmetrised reference
    for r in range(world):
        W, H, g, halo, send = out[r]
        assert np.allclose(W[..., 1:], gu, atol=1e-12) and np.allclose(W[..., 0], gx, atol=1e-12)
        assert np.allclose(0.5 * (H + H.T), H_ref, atol=1e-10)
        assert np.allclose(g, qp.g, atol=1e-10)
    # halo / send lists are mutually consistent
    for r in range(world):
        for p, ids in out[r][3].items():
            assert out[p][4][r] == ids


def test_partition_plan_mesh_row_slabs():
    topo = mesh_topology(8, 5)
    parts = [partition_nodes(topo, 4, r) for r in range(4)]
    assert [p.lo for p in parts] == [0, 10, 20, 30] and parts[-1].hi == 40
    # interior slabs see one boundary row (5 nodes) on each side
    assert sorted(parts[1].halo) == [0, 2]
    assert parts[1].halo[0].tolist() == list(range(5, 10))
    assert parts[1].halo[2].tolist() == list(range(20, 25))
    assert parts[1].send[0].tolist() == list(range(10, 15))
    for p in parts:
        assert set(np.concatenate(list(p.halo.values()))) <= set(range(40)) - set(range(p.lo, p.hi))


def test_shard_range_covers_all_instances():
    for B in (1, 7, 4096):
        for w in (1, 2, 3, 8):
            spans = [shard_range(B, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
