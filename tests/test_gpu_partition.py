"""The node-partitioned RTI step (cfg5 design, partition.py) executed on the
GPU at world sizes 1, 2 and 4 against the CPU oracle.

The box has one GPU, so the ranks run as threads of this process, each with
its own stream and its own native context, talking through the in-process
``LocalTransport`` (device-to-device copies behind a barrier; no kernel ever
waits on another rank's kernel).  Everything else is the production path:
node-range K-LIN on the owned nodes, per-stage ``gm_condense_gammas_stage``
with the halo rows packed / unpacked by ``gm_gather_rows`` /
``gm_scatter_rows``, the partial K-HG (R-bar on rank 0 only), masked
constraint rows, one all-reduce of [H | g | C | d], the replicated QP and
K-RS over owned + halo nodes.

Tolerances as everywhere: u, trajectories
max|d| / max(1, max|ref|) <= 1e-4; status equal, iterations +-1.
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _problem(rows, cols, N, hard=True):
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.condensing import OcpSpec, StateConstraint

    topo, model, states, inputs, spec = workloads.mesh_problem(rows, cols, N, 0.01, 2)
    M = rows * cols
    scons = list(spec.state_constraints)
    if hard:
        # hard rows on nodes spread over the slabs (row masking / ownership)
        for node in (1, M // 3, M // 2 + 1, M - 2):
            c = np.zeros((2, 6))
            c[0, 2], c[1, 0] = 1.0, -1.0
            x = states[0][node]
            for k in (2, N):
                scons.append(StateConstraint(node, k, c, np.array([x[2] + 0.05, -(x[0] - 0.05)])))
    spec = OcpSpec(topo, N, spec.q, spec.x_ref, spec.r, spec.u_ref, spec.input_constraints, scons)
    return topo, model, states, inputs, spec


def _run_ranks(world, topo, model, spec, cfg, x0, ls, li, steps=2, last=None):
    """Run ``steps`` partitioned RTI steps on ``world`` thread-ranks; returns
    per rank [(u, status, iters, next_states_local)] and the partitions."""
    import torch

    from paper_2602_17601_b200.partition import (LocalHub, LocalTransport, PartitionedMpc,
                                                 partition_nodes)

    hub = LocalHub(world)
    parts = [partition_nodes(topo, world, r) for r in range(world)]
    out = {}
    errs = []

    def run(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                pm = PartitionedMpc(model, topo, spec, cfg, parts[r],
                                    transport=LocalTransport(hub, r) if world > 1 else None)
                res = []
                s_ls, s_li, prev = ls, li, last
                for _ in range(steps):
                    u, st, it = pm.step(x0, s_ls, s_li, last_applied=prev)
                    ns = pm.next_states.clone()
                    res.append((u, st, it, ns.cpu().numpy(), pm.next_inputs.cpu().numpy()))
                    s_ls, s_li, prev = ns, pm.next_inputs.clone(), u
                    torch.cuda.current_stream().synchronize()
                out[r] = res
        except BaseException as e:  # pragma: no cover - surfaced below
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    assert not errs, errs
    return out, parts


def _oracle_steps(topo, model, spec, x0, ls, li, N, steps=2):
    from oracle import ref_port as O

    res = []
    last = None
    for _ in range(steps):
        o = O.mpc_step(model, topo, spec, x0, ls, li, N, last_applied=last)
        res.append(o)
        ls, li, last = o["lin_states"], o["lin_inputs"], o["u_applied"]
    return res


@pytest.mark.parametrize("shape,N,worlds", [((12, 10), 8, (1, 2, 4)), ((40, 25), 20, (1, 2, 4))])
def test_partitioned_mpc_matches_oracle(shape, N, worlds):
    """Two RTI steps per world size.  Each step is compared with the oracle's
    step from the SAME controller state (the previous GPU step's plan,
    assembled from the ranks' owned rows), so every step is a one-step
    parity check: a linearisation point that moved by the fp32 round-off of
    the previous step can flip a ReLU mask whose pre-activation sits within
    ~1e-6 of the kink and legitimately change the next QP."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O

    topo, model, states, inputs, spec = _problem(*shape, N)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x0 = states[0]
    M = topo.node_count
    for world in worlds:
        ls, li, last = np.concatenate([states, states[-1:]], 0), inputs, None
        for t in range(2):
            o = O.mpc_step(model, topo, spec, x0, ls, li, N, last_applied=last)
            out, parts = _run_ranks(world, topo, model, spec, cfg, x0, ls, li, steps=1, last=last)
            nxt = np.empty((N + 1, M, 6))
            for r in range(world):
                loc = parts[r].local_nodes
                u, st, it, ns, ni = out[r][0]
                info = (shape, world, r, t)
                assert pkg.qpsolver.STATUS_BY_CODE[st].value == o["status"], info
                assert abs(it - o["iterations"]) <= 1, info
                scale = max(1.0, float(np.max(np.abs(o["u_applied"]))))
                assert float(np.max(np.abs(u - o["u_applied"]))) / scale <= TOL, info
                # the successor trajectory of owned AND halo nodes
                xs = max(1.0, float(np.max(np.abs(o["lin_states"]))))
                assert float(np.max(np.abs(ns - o["lin_states"][:, loc]))) / xs <= TOL, info
                assert float(np.max(np.abs(ni - o["lin_inputs"]))) / scale <= TOL, info
                own = slice(parts[r].own_lo, parts[r].own_hi) if world > 1 else slice(0, M)
                nxt[:, parts[r].lo:parts[r].hi] = ns[:, own]
            # every rank solved the identical all-reduced QP: identical inputs
            for r in range(1, world):
                assert np.array_equal(out[r][0][0], out[0][0][0])
            ls, li, last = nxt, out[0][0][4], out[0][0][0]


def test_partitioned_engines_do_not_leak_node_range():
    """A PartitionedMpc owns a private context: a cached engine on the same
    topology (mpc_step, linearize_trajectory) keeps the whole node range
    while partitioned ranks run (advisor finding, partition.py)."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O

    topo, model, states, inputs, spec = _problem(8, 6, 6, hard=False)
    cfg = pkg.MpcConfig(horizon=6, dt=0.01)
    _run_ranks(2, topo, model, spec, cfg, states[0], np.concatenate([states, states[-1:]], 0),
               inputs, steps=1)
    lin = pkg.linearize_trajectory(model, topo, states, inputs)
    ref = O.linearize_trajectory(model, topo, states, inputs)
    assert np.max(np.abs(lin.a_self - ref.a_self)) / np.max(np.abs(ref.a_self)) <= TOL


def test_halo_gather_scatter_kernels():
    """gm_gather_rows / gm_scatter_rows against torch indexing (strided rows,
    an outer stride for (stage, node)-major trajectories)."""
    import torch

    from paper_2602_17601_b200 import device

    eng = device.engine(device_topo())
    rng = np.random.default_rng(0)
    src = torch.from_numpy(rng.standard_normal((9, 5, 6, 8)).astype(np.float32)).cuda()
    idx = torch.tensor([7, 0, 3, 8], dtype=torch.int32, device="cuda")
    stage = 2
    dst = torch.empty((4, 6, 8), dtype=torch.float32, device="cuda")
    es = src.element_size()
    eng.ctx.call("gm_gather_rows", src.data_ptr() + stage * src.stride(1) * es, dst.data_ptr(),
                 idx.data_ptr(), 4, 6 * 8 * es, src.stride(0) * es, 1, 0, eng.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dst, src[:, stage].index_select(0, idx.long()))
    out = torch.zeros_like(src)
    eng.ctx.call("gm_scatter_rows", dst.data_ptr(), out.data_ptr() + stage * src.stride(1) * es,
                 idx.data_ptr(), 4, 6 * 8 * es, src.stride(0) * es, 1, 0, eng.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out[:, stage].index_select(0, idx.long()), dst)
    # (N+1, M, nx) fp64 trajectory rows of nodes idx across all stages
    traj = torch.from_numpy(rng.standard_normal((5, 9, 6))).cuda()
    d2 = torch.empty((5, 4, 6), dtype=torch.float64, device="cuda")
    es = traj.element_size()
    eng.ctx.call("gm_gather_rows", traj.data_ptr(), d2.data_ptr(), idx.data_ptr(), 4, 6 * es,
                 traj.stride(1) * es, 5, traj.stride(0) * es, eng.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(d2, traj.index_select(1, idx.long()))


def device_topo():
    from paper_2602_17601_b200.graph import chain_topology

    return chain_topology(1)
