"""GPU tests of the batched (cfg4) and node-partitioned (cfg5) step drivers.

Only one GPU is available to the test runner, so the partitioned driver runs
with a world-size-1 NCCL group here (the exchange/reduction logic itself is
covered with 2-3 gloo ranks in tests/test_distributed_cpu.py)."""

import os
import socket

import numpy as np
import pytest

from tests.golden_io import STATUS

pytestmark = pytest.mark.gpu


def test_batched_step_matches_oracle_per_instance():
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.batch import BatchedMpc

    M, N, B = 12, 8, 3
    topo, model, _, _, spec = workloads.scaling_problem(M, N, 0.01, 0)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    xs, ls, li, xr = [], [], [], []
    for b in range(B):
        st, inp = workloads.batch_instance(b, M, N)
        xs.append(st[0])
        ls.append(np.concatenate([st, st[-1:]], axis=0))
        li.append(inp)
        xr.append(np.repeat(st[0][:, None, :], N + 1, axis=1))
    bm = BatchedMpc(model, topo, spec, cfg, B)
    res = bm.step(np.stack(xs), np.stack(ls), np.stack(li), np.stack(xr))
    nxt = res.next_states.cpu().numpy()
    for b in range(B):
        spec_b = pkg.OcpSpec(topo, N, spec.q, xr[b], spec.r, spec.u_ref, spec.input_constraints,
                             spec.state_constraints)
        ref = O.mpc_step(model, topo, spec_b, xs[b], ls[b], li[b], N)
        assert res.status[b].value == ref["status"]
        scale = max(1.0, float(np.max(np.abs(ref["u_applied"]))))
        assert float(np.max(np.abs(res.u_applied[b] - ref["u_applied"]))) / scale <= 1e-4
        assert np.max(np.abs(nxt[b] - ref["lin_states"])) / np.max(np.abs(ref["lin_states"])) <= 1e-4


def test_wave_pipeline_matches_batched_step():
    """WavePipeline (H2D of wave w on a side stream under wave w-1's kernels)
    gives the same per-wave results as BatchedMpc.step, over two passes so
    both buffer sets of each size are reused."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.batch import BatchedMpc, WavePipeline

    M, N = 12, 8
    sizes = [3, 3, 2, 3]
    topo, model, _, _, spec = workloads.scaling_problem(M, N, 0.01, 0)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    waves, i0 = [], 0
    for n in sizes:
        xs, ls, li, xr = [], [], [], []
        for b in range(i0, i0 + n):
            st, inp = workloads.batch_instance(b, M, N)
            xs.append(st[0])
            ls.append(np.concatenate([st, st[-1:]], axis=0))
            li.append(inp)
            xr.append(np.repeat(st[0][:, None, :], N + 1, axis=1))
        waves.append(tuple(torch.from_numpy(np.stack(v)).pin_memory() for v in (xs, ls, li, xr)))
        i0 += n
    ref = [BatchedMpc(model, topo, spec, cfg, n).step(*w) for n, w in zip(sizes, waves)]
    pipe = WavePipeline(model, topo, spec, cfg, sizes)
    for _ in range(2):
        got = pipe.step(waves)
        for r, g in zip(ref, got):
            assert [s.value for s in g.status] == [s.value for s in r.status]
            np.testing.assert_array_equal(g.iterations, r.iterations)
            np.testing.assert_array_equal(g.u_applied, r.u_applied)
            np.testing.assert_array_equal(g.next_states.cpu().numpy(), r.next_states.cpu().numpy())
            np.testing.assert_array_equal(g.next_inputs.cpu().numpy(), r.next_inputs.cpu().numpy())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partitioned_step_world1_matches_single_device():
    import torch
    import torch.distributed as dist

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.partition import PartitionedMpc, partition_nodes

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        topo, model, states, inputs, spec = workloads.mesh_problem(6, 5, 6, 0.01, 0)
        N = 6
        cfg = pkg.MpcConfig(horizon=N, dt=0.01)
        x = pkg.SystemState(states[0])
        st = pkg.mpc_init(x, cfg, 6)
        u_ref, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
        pm = PartitionedMpc(model, topo, spec, cfg, partition_nodes(topo, 1, 0))
        u, status, iters = pm.step(states[0], st.lin_states, st.lin_inputs)
        assert status == ["optimal", "max_iterations", "primal_infeasible",
                          "numerical_failure"].index(st1.last_status.value)
        assert np.max(np.abs(u - u_ref.u)) <= 1e-9 * max(1.0, np.max(np.abs(u_ref.u)))
        assert np.max(np.abs(pm.next_states.cpu().numpy() - st1.lin_states)) <= 1e-9
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["chain", "mesh"])
def test_rollout_epilogue_equals_gamma_epilogue(kind, monkeypatch):
    """K-RS by linear rollout (gm_mpc_finish_rollout, the large-batch path)
    against the Gamma-row K-RS (gm_mpc_finish) on the same solved QPs, and
    both against the oracle (reconstruct_states = rollout:
    reference tests/test_condensing.py:120-135).  fp32 blocks either way:
    trajectories within 1e-5 of each other, 1e-4 of the oracle."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.batch import BatchedMpc

    N, B = 8, 3
    if kind == "chain":
        M = 12
        topo, model, _, _, spec = workloads.scaling_problem(M, N, 0.01, 0)
        inst = [workloads.batch_instance(b, M, N) for b in range(B)]
    else:
        topo, model, states, inputs, spec = workloads.mesh_problem(6, 5, N, 0.01, 0)
        M = topo.node_count
        rng = np.random.default_rng(5)
        inst = [(states + 0.01 * rng.standard_normal(states.shape), inputs) for _ in range(B)]
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    xs = np.stack([st[0] for st, _ in inst])
    ls = np.stack([np.concatenate([st, st[-1:]], axis=0) for st, _ in inst])
    li = np.stack([inp for _, inp in inst])
    xr = np.stack([np.repeat(st[0][:, None, :], N + 1, axis=1) for st, _ in inst])
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("GM_FIN_ROLLOUT", mode)
        bm = BatchedMpc(model, topo, spec, cfg, B)
        res = bm.step(xs, ls, li, xr)
        out[mode] = (res, res.next_states.cpu().numpy(), bm.planned_states.cpu().numpy())
    (r0, n0, p0), (r1, n1, p1) = out["0"], out["1"]
    assert np.array_equal(r0.u_applied, r1.u_applied)
    assert [s.value for s in r0.status] == [s.value for s in r1.status]
    scale = np.max(np.abs(n0))
    assert np.max(np.abs(n1 - n0)) / scale <= 1e-5
    assert np.max(np.abs(p1 - p0)) / scale <= 1e-5
    for b in range(B):
        spec_b = pkg.OcpSpec(topo, N, spec.q, xr[b], spec.r, spec.u_ref, spec.input_constraints,
                             spec.state_constraints)
        ref = O.mpc_step(model, topo, spec_b, xs[b], ls[b], li[b], N)
        assert r1.status[b].value == ref["status"]
        assert np.max(np.abs(n1[b] - ref["lin_states"])) / np.max(np.abs(ref["lin_states"])) <= 1e-4


def test_rollout_epilogue_rejects_node_range_and_dims():
    """The rollout entry point fails loudly outside its domain."""
    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime, workloads
    from paper_2602_17601_b200.device import engine

    topo, model, _, _, _ = workloads.scaling_problem(12, 4, 0.01, 0)
    eng = engine(topo, model)
    ctx = eng.ctx
    ctx.call("gm_set_node_range", 2, 8)
    try:
        with pytest.raises(Exception):
            ctx.call("gm_mpc_finish_rollout", 1, 4, None, None, None, None, None, None, 24,
                     None, None, None, None, None, None, 1.0, 0, None, 0, None, None, None,
                     None, None, None, None, None)
    finally:
        ctx.call("gm_set_node_range", 0, 12)


def test_rollout_epilogue_abi_statuses_and_damping():
    """gm_mpc_finish_rollout against gm_mpc_finish through the C ABI on the
    same synthetic blocks, solution and statuses (optimal / primal infeasible
    -> fallback plan / max iterations), with damping 0.5 and the
    hold-previous-input fallback: identical inputs, identical fallback rows,
    planned / shifted trajectories within fp32 block rounding."""
    import torch

    from paper_2602_17601_b200 import device as dev
    from paper_2602_17601_b200._runtime import lib
    from paper_2602_17601_b200.graph import mesh_topology

    topo = mesh_topology(7, 5)
    M, N, B, nx, nu = topo.node_count, 6, 3, 6, 6
    eng = dev.engine(topo)
    eng.set_dims(nx, nu)
    rng = np.random.default_rng(17)
    E = eng.E
    f32, f64 = np.float32, np.float64
    a_self = eng.h2d((rng.standard_normal((B * N, M, nx, nx)) * 0.2 + np.eye(nx) * 0.9).astype(f32), f32)
    a_nbr = eng.h2d((rng.standard_normal((B * N, E, nx, nx)) * 0.1).astype(f32), f32)
    b = eng.h2d(rng.standard_normal((B * N, M, nx, nu)).astype(f32), f32)
    c = eng.h2d(rng.standard_normal((B * N, M, nx)) * 0.1, f64)
    x0 = eng.h2d(rng.standard_normal((B, M, nx)), f64)
    ld = lib().gm_gamma_ld(N, nu)
    W = eng.zeros((B, M, N + 1, nx, ld), f32)
    sp = eng.stream_ptr()
    eng.ctx.call("gm_condense_gammas", B, N, a_self.data_ptr(), a_nbr.data_ptr(), b.data_ptr(), c.data_ptr(),
                 x0.data_ptr(), W.data_ptr(), ld, sp)
    n = N * nu + 4  # solution rows carry trailing slacks like the expanded QP
    u = eng.h2d(rng.standard_normal((B, n)) * 0.3, f64)
    status = torch.tensor([0, 2, 1], dtype=torch.int32, device=u.device)
    iters = torch.tensor([7, 9, 50], dtype=torch.int32, device=u.device)
    lin_s = eng.h2d(rng.standard_normal((B, N + 1, M, nx)), f64)
    lin_u = eng.h2d(rng.standard_normal((B, N, nu)), f64)
    fb_s = eng.h2d(rng.standard_normal((B, N + 1, M, nx)), f64)
    fb_u = eng.h2d(rng.standard_normal((B, N, nu)), f64)
    u_prev = eng.h2d(rng.standard_normal((B, nu)), f64)

    def outs():
        return [eng.zeros(s, f64) for s in ((B, N + 1, M, nx), (B, M, N + 1, nx), (B, N, nu), (B, N + 1, M, nx),
                                            (B, N, nu), (B, nu), (B, nu + 2))]

    def tail(o):
        return (status.data_ptr(), iters.data_ptr(), lin_s.data_ptr(), lin_u.data_ptr(), fb_s.data_ptr(),
                fb_u.data_ptr(), 0.5, 0, u_prev.data_ptr(), 1, *[t.data_ptr() for t in o], sp)

    o1, o2 = outs(), outs()
    eng.ctx.call("gm_mpc_finish", B, N, W.data_ptr(), ld, u.data_ptr(), n, *tail(o1))
    eng.ctx.call("gm_mpc_finish_rollout", B, N, a_self.data_ptr(), a_nbr.data_ptr(), b.data_ptr(), c.data_ptr(),
                 x0.data_ptr(), u.data_ptr(), n, *tail(o2))
    torch.cuda.synchronize()
    r1, r2 = [[t.cpu().numpy() for t in o] for o in (o1, o2)]
    for k in (2, 4, 5, 6):  # inputs, u_applied, summary: no Gamma involved -> identical
        assert np.array_equal(r1[k], r2[k]), k
    fb = fb_s.cpu().numpy()
    for k in (0, 3):  # cur / next states: the failed instance takes the fallback plan exactly
        assert np.array_equal(r1[k][1], r2[k][1])
    assert np.array_equal(r2[0][1], fb[1])
    for k in (0, 1, 3):
        scale = np.max(np.abs(r1[k]))
        assert np.max(np.abs(r1[k] - r2[k])) / scale <= 1e-5, k
