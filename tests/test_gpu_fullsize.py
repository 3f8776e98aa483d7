"""Full-size parity: the cfg3 workload (chain M=1000, N=20, the paper's 100 Hz
headline) on the GPU against the CPU oracle on the same seeded inputs, and
size-independent properties at the larger configs."""

import numpy as np
import pytest

from tests.golden_io import rel

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def cfg3():
    from oracle import ref_port as O
    from paper_2602_17601_b200 import workloads

    topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
    lin = O.linearize_trajectory(model, topo, states, inputs)
    gu, gx = O.condense_gammas(lin, states[0])
    qp = O.condense_ocp(spec, lin, states[0], gammas=(gu, gx))
    H, g, C, d, n0 = O.expand_soft_constraints(qp)
    sol = O.solve_qp(H, g, C, d)
    return dict(topo=topo, model=model, states=states, inputs=inputs, spec=spec, lin=lin, gu=gu,
                gx=gx, qp=qp, sol=sol, n0=n0)


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_cfg3_stages(cfg3, mode):
    """mode 1: fused per-tile linearisation, 2: layer-wise with fused chains
    (forward on fp64 DMMA, Jacobians on tcgen05), 3: per-layer GEMM chain,
    4: as 2 with the per-row SIMT chains."""
    import paper_2602_17601_b200 as pkg

    c = cfg3
    ctx = pkg.device.engine(c["topo"], c["model"]).ctx
    ctx.call("gm_set_linearize_mode", mode)
    try:
        lin = pkg.linearize_trajectory(c["model"], c["topo"], c["states"], c["inputs"])
    finally:
        ctx.call("gm_set_linearize_mode", 0)
    for k in ("a_self", "a_nbr", "b"):
        assert rel(getattr(lin, k), getattr(c["lin"], k)) <= TOL, k
    assert np.max(np.abs(lin.c - c["lin"].c)) / np.max(np.abs(c["states"])) <= TOL
    gu, gx = pkg.condense_gammas(lin, c["states"][0])
    assert rel(gu, c["gu"]) <= TOL
    assert rel(gx, c["gx"]) <= TOL
    qp = pkg.condense_ocp(c["spec"], lin, c["states"][0], gammas=(gu, gx))
    assert rel(qp.h, c["qp"].h) <= TOL
    assert rel(qp.g, c["qp"].g) <= TOL
    assert rel(qp.c, c["qp"].c) <= TOL


def test_cfg3_mpc_step_u0(cfg3):
    import paper_2602_17601_b200 as pkg

    c = cfg3
    N = 20
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(c["states"][0])
    st = pkg.mpc_init(x, cfg, 6)
    st.lin_states = np.concatenate([c["states"], c["states"][-1:]], axis=0)
    st.lin_inputs = c["inputs"]
    u, st1 = pkg.mpc_step(c["model"], c["topo"], c["spec"], x, st, cfg)
    from oracle import ref_port as O

    ref = O.mpc_step(c["model"], c["topo"], c["spec"], c["states"][0], st.lin_states,
                     st.lin_inputs, N)
    assert st1.last_status.value == ref["status"]
    scale = max(1.0, float(np.max(np.abs(ref["u_applied"]))))
    assert float(np.max(np.abs(u.u - ref["u_applied"]))) / scale <= TOL
    assert rel(st1.planned_inputs, ref["planned_inputs"]) <= TOL


def test_many_state_constraints_at_scale():
    """state constraints on many nodes make the QP's general
    rows dominate (m >> 280).  Chain M=400, N=20, hard rows on every 20th
    node at every stage (one upper bound on the height z, one lower bound on
    the lateral position x, the second one active for a few nodes):
    m = 240 box + 800 general rows, n = 120.  condense_ocp's constraint rows
    and the mpc_step input against the CPU oracle (condensing.py:263-282,
    qpsolver.py:112-243); the general rows no longer fit on chip and stream
    from the QP workspace."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.condensing import OcpSpec, StateConstraint

    M, N = 400, 20
    topo, model, states, inputs, spec0 = workloads.scaling_problem(M, N, 0.01, 3)
    rows = []
    for node in range(0, M, 20):
        cz = np.zeros((2, 6))
        cz[0, 2] = 1.0    # z <= z0 + 0.05
        cz[1, 0] = -1.0   # x >= x0 + (0.002 on a few nodes: active)
        for k in range(1, N + 1):
            x0 = states[0][node]
            d = np.array([x0[2] + 0.05, -(x0[0] + (0.002 if node % 100 == 0 else -0.05))])
            rows.append(StateConstraint(node, k, cz, d, soft=False))
    spec = OcpSpec(topo, N, spec0.q, spec0.x_ref, spec0.r, spec0.u_ref, spec0.input_constraints, rows)

    lin = O.linearize_trajectory(model, topo, states, inputs)
    qref = O.condense_ocp(spec, lin, states[0])
    linb = pkg.linearize_trajectory(model, topo, states, inputs)
    qb = pkg.condense_ocp(spec, linb, states[0])
    assert qb.c.shape == qref.c.shape and qb.c.shape[0] == 240 + 2 * 20 * N
    assert rel(qb.c, qref.c) <= TOL
    assert rel(qb.d, qref.d) <= TOL

    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(states[0])
    st = pkg.mpc_init(x, cfg, 6)
    st.lin_states = np.concatenate([states, states[-1:]], axis=0)
    st.lin_inputs = inputs
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
    ref = O.mpc_step(model, topo, spec, states[0], st.lin_states, st.lin_inputs, N)
    assert st1.last_status.value == ref["status"]
    if ref["status"] == "optimal":
        scale = max(1.0, float(np.max(np.abs(ref["u_applied"]))))
        assert float(np.max(np.abs(u.u - ref["u_applied"]))) / scale <= TOL


def _spec_with_r(spec, r_scale):
    from paper_2602_17601_b200.condensing import OcpSpec

    N = spec.horizon
    return OcpSpec(spec.topology, N, spec.q, spec.x_ref, np.tile(np.eye(6) * r_scale, (N, 1, 1)),
                   spec.u_ref, spec.input_constraints, spec.state_constraints)


@pytest.mark.parametrize("r_scale", [10.0, 100.0])
def test_cfg3_interior_qp_u(cfg3, r_scale):
    """An interior-solution QP at the headline size (SURVEY 8c instance P4 at
    M=1000): with R = r_scale * I, 11 (R=10) / 56 (R=100) of the 120 optimal
    inputs lie strictly inside the box, so the fp32 Gamma/H error reaches u.
    Every planned input (not only u0) against the oracle's warm-started solve
    of the same QP: max|du| / max(1, max|u|) <= 1e-4."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O

    c = cfg3
    N = 20
    spec = _spec_with_r(c["spec"], r_scale)
    qp = O.condense_ocp(spec, c["lin"], c["states"][0], gammas=(c["gu"], c["gx"]))
    H, g, C, d, n0 = O.expand_soft_constraints(qp)
    warm = np.zeros(H.shape[0])
    warm[:n0] = c["inputs"].reshape(-1)
    sol = O.solve_qp(H, g, C, d, warm_start=warm)
    u_ref = sol.u[:n0]
    interior = int(np.sum((u_ref > 1e-6) & (u_ref < 8 - 1e-6)))
    assert interior >= 10
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(c["states"][0])
    st = pkg.mpc_init(x, cfg, 6)
    st.lin_states = np.concatenate([c["states"], c["states"][-1:]], axis=0)
    st.lin_inputs = c["inputs"]
    u, st1 = pkg.mpc_step(c["model"], c["topo"], spec, x, st, cfg)
    assert st1.last_status.value == sol.status
    assert abs(st1.last_iterations - sol.iterations) <= 1
    scale = max(1.0, float(np.max(np.abs(u_ref))))
    assert float(np.max(np.abs(st1.planned_inputs.reshape(-1) - u_ref))) / scale <= TOL
    assert float(np.max(np.abs(u.u - u_ref[:6]))) / scale <= TOL


@pytest.fixture(scope="module")
def mesh100():
    """The cfg5 recipe on a 100 x 100 mesh (M = 10^4, E = 39,600, degree 4),
    N = 20: the oracle's blocks, Gammas, H, g (about 20 s of CPU)."""
    from oracle import ref_port as O
    from paper_2602_17601_b200 import workloads

    topo, model, states, inputs, spec = workloads.mesh_problem(100, 100, 20, 0.01, 0)
    lin = O.linearize_trajectory(model, topo, states, inputs)
    gu, gx = O.condense_gammas(lin, states[0], threads=8)
    return dict(topo=topo, model=model, states=states, inputs=inputs, spec=spec, lin=lin, gu=gu,
                gx=gx)


def test_mesh_fullsize_stages(mesh100):
    """Degree-4 psi aggregation and the 5-block neighbour recursion at 10^4
    nodes against the oracle: A, B, c, Gamma_u, Gamma_x, H, g, C, d."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O

    c = mesh100
    lin = pkg.linearize_trajectory(c["model"], c["topo"], c["states"], c["inputs"])
    for k in ("a_self", "a_nbr", "b"):
        assert rel(getattr(lin, k), getattr(c["lin"], k)) <= TOL, k
    assert np.max(np.abs(lin.c - c["lin"].c)) / np.max(np.abs(c["states"])) <= TOL
    gu, gx = pkg.condense_gammas(lin, c["states"][0])
    assert rel(gu, c["gu"]) <= TOL
    assert rel(gx, c["gx"]) <= TOL
    qref = O.condense_ocp(c["spec"], c["lin"], c["states"][0], gammas=(c["gu"], c["gx"]), threads=8)
    qp = pkg.condense_ocp(c["spec"], lin, c["states"][0])
    assert rel(qp.h, qref.h) <= TOL
    assert rel(qp.g, qref.g) <= TOL
    assert rel(qp.c, qref.c) <= TOL
    assert float(np.max(np.abs(qp.d - qref.d))) <= TOL * max(1.0, float(np.max(np.abs(qref.d))))


@pytest.mark.parametrize("r_scale", [0.01, 1.0])
def test_mesh_fullsize_mpc_step(mesh100, r_scale):
    """mpc_step at 10^4 mesh nodes: the default spec (R = 0.01 I, bang-bang)
    and R = I (interior inputs) against the oracle's warm-started solve."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O

    c = mesh100
    N = 20
    spec = _spec_with_r(c["spec"], r_scale)
    qp = O.condense_ocp(spec, c["lin"], c["states"][0], gammas=(c["gu"], c["gx"]), threads=8)
    H, g, C, d, n0 = O.expand_soft_constraints(qp)
    warm = np.zeros(H.shape[0])
    warm[:n0] = c["inputs"].reshape(-1)
    sol = O.solve_qp(H, g, C, d, warm_start=warm)
    u_ref = sol.u[:n0]
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(c["states"][0])
    st = pkg.mpc_init(x, cfg, 6)
    st.lin_states = np.concatenate([c["states"], c["states"][-1:]], axis=0)
    st.lin_inputs = c["inputs"]
    u, st1 = pkg.mpc_step(c["model"], c["topo"], spec, x, st, cfg)
    assert st1.last_status.value == sol.status
    scale = max(1.0, float(np.max(np.abs(u_ref))))
    assert float(np.max(np.abs(st1.planned_inputs.reshape(-1) - u_ref))) / scale <= TOL
    assert float(np.max(np.abs(u.u - u_ref[:6]))) / scale <= TOL
