"""Multi-rank host logic on CPU (gloo world_size 2 and 3; the in-process
thread transport at 2-4 ranks).

The node-partitioned condensing (paper_2602_17601_b200/partition.py) is run
with the real partition plan (local owned + halo numbering), the real
point-to-point halo exchange and the real all-reduce; the per-rank stage
update is a NumPy restatement of K-REC restricted to owned nodes.  Every local
Gamma row (halo included) and the all-reduced H/g must equal the
single-process oracle (condensing.py:182-228, :363-406).  The same partition
code runs the GPU kernels in tests/test_gpu_partition.py.
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
from paper_2602_17601_b200.partition import (DistTransport, HaloExchange, LocalHub,
                                             LocalTransport, partition_nodes)


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


def _rank_condense(part, transport, topo, N=4, nx=2, nu=1):
    """One rank of the partitioned recursion + cost on its local graph
    (owned + halo rows), with the real halo exchange and the real
    all-reduce; the per-rank stage update is a NumPy restatement of K-REC
    restricted to owned nodes (condensing.py:211-224)."""
    lin, spec, x0 = _instance(topo, N, nx, nu)
    ltopo = part.local_topology(topo)
    ML = ltopo.node_count
    loc = part.local_nodes
    lptr, lsrc = ltopo.csr()
    gptr, _ = topo.csr()
    W = torch.zeros((ML, N + 1, nx, 1 + N * nu), dtype=torch.float64)
    W[:, 0, :, 0] = torch.from_numpy(x0[loc])
    halo = HaloExchange(part, W, transport, torch_pack=True)
    for n in range(N):
        live = 1 + n * nu
        prev = W[:, n].numpy()
        for li in range(part.own_lo, part.own_hi):
            gi = int(loc[li])
            acc = lin.a_self[n, gi] @ prev[li, :, :live]
            for k, e in enumerate(range(lptr[li], lptr[li + 1])):
                ge = gptr[gi] + k  # same in-edge order in the local graph
                acc = acc + lin.a_nbr[n, ge] @ prev[lsrc[e], :, :live]
            acc[:, 0] += lin.c[n, gi]
            W[li, n + 1, :, :live] = torch.from_numpy(acc)
            W[li, n + 1, :, live:live + nu] = torch.from_numpy(lin.b[n, gi])
        halo.exchange(n + 1)
    Wn = W.numpy()
    gu, gx = Wn[..., 1:], Wn[..., 0]
    # partial cost over owned nodes, R-bar on rank 0 only, then all-reduce
    q_lin = -2.0 * np.einsum("mkab,mkb->mka", spec.q, spec.x_ref)
    H = np.zeros((N * nu, N * nu))
    g = np.zeros(N * nu)
    if part.rank == 0:
        H, gr = O.r_bar(spec)
        g = gr.copy()
    own = slice(part.own_lo, part.own_hi)
    gsl = slice(part.lo, part.hi)
    for k in range(1, N + 1):
        Gk = gu[own, k, :, : k * nu]
        H[: k * nu, : k * nu] += np.tensordot(Gk, spec.q[gsl, k] @ Gk, axes=([0, 1], [0, 1]))
        wk = 2.0 * (spec.q[gsl, k] @ gx[own, k, :, None])[..., 0] + q_lin[gsl, k]
        g[: k * nu] += np.einsum("mab,ma->b", Gk, wk)
    red = torch.from_numpy(np.concatenate([H.ravel(), g]))
    transport.allreduce_sum(red)
    red = red.numpy()
    return (Wn.copy(), red[: H.size].reshape(H.shape), red[H.size:],
            {p: v.tolist() for p, v in part.halo.items()},
            {p: v.tolist() for p, v in part.send.items()}, loc.copy())


def _worker(rank, world, port, graph, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        topo = chain_topology(11) if graph == "chain" else mesh_topology(5, 4)
        part = partition_nodes(topo, world, rank)
        out[rank] = _rank_condense(part, DistTransport(), topo)
    finally:
        dist.destroy_process_group()


def _check(topo, world, out):
    lin, spec, x0 = _instance(topo)
    gu, gx = O.condense_gammas(lin, x0)
    qp = O.condense_ocp(spec, lin, x0, gammas=(gu, gx))
    for r in range(world):
        W, H, g, halo, send, loc = out[r]
        # every local row (owned AND halo) equals the single-process Gammas
        assert np.allclose(W[..., 1:], gu[loc], atol=1e-12)
        assert np.allclose(W[..., 0], gx[loc], atol=1e-12)
        assert np.allclose(0.5 * (H + H.T), qp.h, atol=1e-10)
        assert np.allclose(g, qp.g, atol=1e-10)
    # halo / send lists are mutually consistent
    for r in range(world):
        for p, ids in out[r][3].items():
            assert out[p][4][r] == ids


@pytest.mark.parametrize("graph,world", [("chain", 2), ("mesh", 2), ("mesh", 3)])
def test_partitioned_condensing_matches_single_process(graph, world):
    """gloo, one process per rank (the torch.distributed transport)."""
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
    _check(topo, world, dict(out))


@pytest.mark.parametrize("graph,world", [("chain", 3), ("mesh", 2), ("mesh", 4)])
def test_partitioned_condensing_local_transport(graph, world):
    """The in-process transport (ranks as threads) used by the one-GPU
    partition tests gives the same result as gloo / the single process."""
    import threading

    topo = chain_topology(11) if graph == "chain" else mesh_topology(5, 4)
    hub = LocalHub(world)
    out, errs = {}, []

    def run(r):
        try:
            out[r] = _rank_condense(partition_nodes(topo, world, r), LocalTransport(hub, r), topo)
        except BaseException as e:  # pragma: no cover - surfaced below
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errs, errs
    _check(topo, world, out)


def test_local_graph_renumbering():
    """Owned nodes are the contiguous local range [own_lo, own_hi); halo
    nodes keep ascending global order and have no in-edges; owned nodes keep
    their in-neighbour order (graph.py:60-63 edge order)."""
    topo = mesh_topology(6, 5)
    for world in (2, 3, 4):
        for r in range(world):
            p = partition_nodes(topo, world, r)
            lt = p.local_topology(topo)
            loc = p.local_nodes
            assert np.all(np.diff(loc) > 0)
            assert loc[p.own_lo:p.own_hi].tolist() == list(range(p.lo, p.hi))
            for li, g in enumerate(loc):
                if p.lo <= g < p.hi:
                    assert [int(loc[j]) for j in lt.in_neighbors[li]] == list(topo.in_neighbors[g])
                else:
                    assert lt.in_neighbors[li] == ()
            halo = sorted(int(v) for ids in p.halo.values() for v in ids)
            assert sorted(set(loc.tolist()) - set(range(p.lo, p.hi))) == halo


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
