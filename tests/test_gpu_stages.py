"""GPU parity of every hot-path stage against the reference's golden vectors
and the CPU oracle (oracle/ref_port.py).

Tolerances (fp32 stages vs the fp64 reference):
  index tables                         bit-exact
  a_self, a_nbr, b, Gamma, H, g, C, d  rel = max|x - ref| / max|ref| <= 1e-4
  c                                     max|dc| / max|x_hat| <= 1e-4
  QP on identical fp64 data (K-QP)     |du| <= 1e-6 (reference tests' own bound)
  u* through the whole pipeline        max|du| / max(1, max|u|) <= 1e-4
"""

from types import SimpleNamespace

import numpy as np
import pytest

from tests.golden_io import (STATUS, mpc_branch_cases, pipeline_case, qp_round2,
                             random_condense_cases, random_qps, rel)

pytestmark = pytest.mark.gpu

TOL = 1e-4
# chains (cfg1 recipe, P3 biases + normalisation, P4 interior QP) and
# 4-neighbour meshes (cfg5 recipe 6x5, P3-style 4x4 with hard + soft rows)
CASES = ["cfg1_chain10", "p3_biases_norm", "p4_interior", "mesh6x5", "mesh_p3"]


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_17601_b200 as p

    return p


def _set_lin_mode(pkg, cs, mode):
    """Force the fused (1), layer-wise with fused chains (2: forward on fp64
    DMMA, Jacobians on tcgen05), fully layer-wise (3) or layer-wise with the
    per-row SIMT chains (4) linearisation kernels; 0 = auto."""
    pkg.device.engine(cs.topo, cs.model).ctx.call("gm_set_linearize_mode", mode)


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_linearize_matches_reference(pkg, name, mode):
    cs = pipeline_case(name)
    _set_lin_mode(pkg, cs, mode)
    try:
        lin = pkg.linearize_trajectory(cs.model, cs.topo, cs.states, cs.inputs)
    finally:
        _set_lin_mode(pkg, cs, 0)
    assert lin.on_device
    d = cs.d
    for k in ("a_self", "a_nbr", "b"):
        assert rel(getattr(lin, k), d["lin_" + k]) <= TOL, k
    xscale = max(1.0, float(np.max(np.abs(cs.states))))
    assert float(np.max(np.abs(lin.c - d["lin_c"]))) / xscale <= TOL


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_affine_model_exact_at_point(pkg, name, mode):
    """x+ = A x + sum A_nbr x_j + B u + c reproduces step_array (gnn.py:291-297)."""
    cs = pipeline_case(name)
    N = cs.inputs.shape[0]
    _set_lin_mode(pkg, cs, mode)
    try:
        lin = pkg.linearize_trajectory(cs.model, cs.topo, cs.states, cs.inputs)
    finally:
        _set_lin_mode(pkg, cs, 0)
    X = cs.states[:N]
    f = pkg.step_array(cs.model, cs.topo, X, cs.inputs)
    rec = np.einsum("kiab,kib->kia", lin.a_self, X) + np.einsum("kiab,kb->kia", lin.b, cs.inputs) + lin.c
    for e, (i, j) in enumerate(cs.topo.edges):
        rec[:, i] += np.einsum("kab,kb->ka", lin.a_nbr[:, e], X[:, j])
    assert np.max(np.abs(rec - f)) <= 1e-9 * max(1.0, np.max(np.abs(f)))


def test_step_array_matches_reference_forward(pkg):
    from oracle import ref_port as O

    cs = pipeline_case("p3_biases_norm")
    f = pkg.step_array(cs.model, cs.topo, cs.states, np.vstack([cs.inputs, cs.inputs[:1]]))
    ref = O.step_array(cs.model, cs.topo, cs.states, np.vstack([cs.inputs, cs.inputs[:1]]))
    assert np.max(np.abs(f - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("name", CASES)
def test_condense_pipeline_matches_reference(pkg, name):
    cs = pipeline_case(name)
    d = cs.d
    lin = pkg.linearize_trajectory(cs.model, cs.topo, cs.states, cs.inputs)
    gu, gx = pkg.condense_gammas(lin, cs.x0)
    assert rel(gu, d["gamma_u"]) <= TOL
    assert rel(gx, d["gamma_x"]) <= TOL
    qp = pkg.condense_ocp(cs.spec, lin, cs.x0, gammas=(gu, gx))
    assert rel(qp.h, d["qp_h"]) <= TOL
    assert rel(qp.g, d["qp_g"]) <= TOL
    assert np.array_equal(qp.h, qp.h.T)
    assert qp.c.shape == d["qp_c"].shape
    if qp.c.size:
        assert rel(qp.c, d["qp_c"]) <= TOL
        assert float(np.max(np.abs(qp.d - d["qp_d"]))) <= TOL * max(1.0, np.max(np.abs(d["qp_d"])))
    assert np.array_equal(qp.soft, d["qp_soft"])


@pytest.mark.parametrize("case", range(12))
def test_random_condense_instances(pkg, case):
    """Reference test-generator instances (tests/test_condensing.py:40-80):
    arbitrary nx, nu, N, degree <= 2, input + state constraints."""
    cs = random_condense_cases()[case]
    gu, gx = pkg.condense_gammas(cs.lin, cs.x0)
    assert rel(gu, cs.gamma_u) <= TOL
    assert rel(gx, cs.gamma_x) <= TOL
    qp = pkg.condense_ocp(cs.spec, cs.lin, cs.x0)
    assert rel(qp.h, cs.qp["h"]) <= TOL
    assert rel(qp.g, cs.qp["g"]) <= TOL
    assert qp.c.shape == cs.qp["c"].shape
    if qp.c.size:
        assert rel(qp.c, cs.qp["c"]) <= TOL
    assert np.array_equal(qp.soft, cs.qp["soft"])


def test_gamma_hand_example(pkg):
    """x_{k+1} = 2 x_k + u_k from x0 = 1 (tests/test_condensing.py:83-88)."""
    topo = pkg.GraphTopology(1, ((),), 1)
    lin = pkg.LinearizedDynamics(topo, 2, np.full((2, 1, 1, 1), 2.0), np.zeros((2, 0, 1, 1)),
                                 np.full((2, 1, 1, 1), 1.0), np.zeros((2, 1, 1)))
    gu, gx = pkg.condense_gammas(lin, np.array([[1.0]]))
    assert np.array_equal(gu[0].reshape(3, 2), [[0, 0], [1, 0], [2, 1]])
    assert np.array_equal(gx[0].reshape(3), [1, 2, 4])


def test_expand_soft_matches_reference(pkg):
    cs = pipeline_case("cfg1_chain10")
    d = cs.d
    qp = pkg.CondensedQp(d["qp_h"], d["qp_g"], d["qp_c"], d["qp_d"], d["qp_soft"], d["qp_rho1"],
                         d["qp_rho2"])
    H, g, C, dd, n0 = pkg.expand_soft_constraints(qp)
    assert n0 == d["qp_h"].shape[0]
    assert np.array_equal(H, d["x_H"]) and np.array_equal(g, d["x_g"])
    assert np.array_equal(C, d["x_C"]) and np.array_equal(dd, d["x_d"])


@pytest.mark.parametrize("name", CASES)
def test_qp_on_reference_data(pkg, name):
    """K-QP on the reference's own expanded QP: same status, same iterations
    (+-1), same u*."""
    cs = pipeline_case(name)
    d = cs.d
    sol = pkg.solve_qp(pkg.QpProblem(d["x_H"], d["x_g"], d["x_C"], d["x_d"]))
    assert sol.status.value == STATUS[int(d["sol_meta"][0])]
    assert abs(sol.iterations - int(d["sol_meta"][1])) <= 1
    scale = max(1.0, float(np.max(np.abs(d["sol_u"]))))
    assert float(np.max(np.abs(sol.u - d["sol_u"]))) / scale <= 1e-6


def test_random_qps(pkg):
    for t, q in enumerate(random_qps()):
        sol = pkg.solve_qp(pkg.QpProblem(q.H, q.g, q.C, q.d))
        info = (t, q.H.shape, q.C.shape, sol.status.value, q.status, sol.iterations, q.iterations,
                float(np.max(np.abs(sol.u - q.u))))
        assert sol.status.value == q.status, info
        assert abs(sol.iterations - q.iterations) <= 1, info
        assert np.max(np.abs(sol.u - q.u)) <= 1e-6, info


def test_qp_batched_matches_single(pkg):
    """Eight same-shape reference QPs (n=5, m=7) in one batched launch (one
    CTA each) against the reference's solutions and the single-QP path."""
    qs = qp_round2().batch
    sols = pkg.solve_qp_batched(np.stack([q.H for q in qs]), np.stack([q.g for q in qs]),
                                np.stack([q.C for q in qs]), np.stack([q.d for q in qs]))
    for t, (q, s) in enumerate(zip(qs, sols)):
        assert s.status.value == q.status, t
        assert abs(s.iterations - q.iterations) <= 1, t
        assert np.max(np.abs(s.u - q.u)) <= 1e-6, t
        one = pkg.solve_qp(pkg.QpProblem(q.H, q.g, q.C, q.d))
        assert np.array_equal(one.u, s.u) and one.iterations == s.iterations, t


def test_qp_best_iterate_at_cap(pkg):
    """The iteration cap returns the best iterate found (qpsolver.py:231-235,
    reference tests/test_qpsolver.py:127-134): caps 1, 2, 3, 5 against the
    reference's own returned iterate."""
    for t, q in enumerate(qp_round2().cap):
        s = pkg.solve_qp(pkg.QpProblem(q.H, q.g, q.C, q.d),
                         pkg.SolverSettings(max_iterations=q.cap))
        assert s.status.value == q.status, (t, s.status, q.status)
        assert s.iterations == q.iterations, t
        assert np.all(np.isfinite(s.u))
        assert np.max(np.abs(s.u - q.u)) <= 1e-9 * max(1.0, np.max(np.abs(q.u))), t


def test_qp_known_answers(pkg):
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.array([-2.0]), np.zeros((0, 1)), np.zeros(0)))
    assert s.status == pkg.QpStatus.OPTIMAL and abs(s.u[0] - 1.0) <= 1e-12
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.array([-2.0]), np.array([[1.0]]), np.array([0.5])))
    assert s.status == pkg.QpStatus.OPTIMAL
    assert abs(s.u[0] - 0.5) <= 1e-7 and abs(s.duals[0] - 1.0) <= 1e-6
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.zeros(1), np.array([[1.0], [-1.0]]),
                                   np.array([-1.0, -2.0])))
    # the reference returns PRIMAL_INFEASIBLE after 6 iterations with the best
    # iterate u = 0 (fixture qp_round2, qpsolver.py:163-165)
    q2 = qp_round2()
    assert s.status.value == q2.infeas_status == "primal_infeasible"
    assert s.iterations == q2.infeas_iterations
    assert np.array_equal(s.u, q2.infeas_u)
    assert abs(s.primal_infeas - q2.infeas_primal) <= 1e-12


@pytest.mark.parametrize("name", CASES)
def test_reconstruct_matches_reference(pkg, name):
    cs = pipeline_case(name)
    d = cs.d
    n0 = d["gamma_u"].shape[-1]
    x = pkg.reconstruct_states(d["gamma_u"], d["gamma_x"], d["sol_u"][:n0])
    assert rel(x, d["recon"]) <= 1e-6


@pytest.mark.parametrize("name", CASES)
def test_mpc_step_matches_reference(pkg, name):
    cs = pipeline_case(name)
    d = cs.d
    N = cs.spec.horizon
    cfg = pkg.MpcConfig(horizon=N, dt=cs.model.dt)
    x = pkg.SystemState(cs.x0)
    st = pkg.mpc_init(x, cfg, cs.spec.n_u)
    u1, st1 = pkg.mpc_step(cs.model, cs.topo, cs.spec, x, st, cfg)
    assert st1.last_status.value == STATUS[int(d["mpc_meta"][0])]
    scale = max(1.0, float(np.max(np.abs(d["mpc_u"]))))
    assert float(np.max(np.abs(u1.u - d["mpc_u"]))) / scale <= TOL
    assert rel(st1.lin_states, d["mpc_lin_states"]) <= TOL
    assert rel(st1.planned_states, d["mpc_planned_states"]) <= TOL
    u2, st2 = pkg.mpc_step(cs.model, cs.topo, cs.spec, x, st1, cfg)
    assert st2.last_status.value == STATUS[int(d["mpc2_meta"][0])]
    assert float(np.max(np.abs(u2.u - d["mpc2_u"]))) / scale <= TOL
    assert rel(st2.lin_states, d["mpc2_lin_states"]) <= TOL


@pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 31, 32, 33, 64, 70, 100, 140, 141, 160])
def test_device_cholesky_and_solve(pkg, n):
    """K-QP's factorisation (2x2-pivot block elimination -> Cholesky) and its
    blocked triangular solves against NumPy on SPD matrices."""
    import torch

    from paper_2602_17601_b200 import device

    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    A = A @ A.T + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    eng = device.engine(pkg.chain_topology(1))
    dA, db = eng.h2d(A, np.float64), eng.h2d(b, np.float64)
    L = eng.empty((n, n), np.float64)
    x = eng.empty((n,), np.float64)
    ok = eng.empty((1,), np.int32)
    eng.ctx.call("gm_chol_check", n, dA.data_ptr(), db.data_ptr(), L.data_ptr(), x.data_ptr(),
                 ok.data_ptr(), eng.stream_ptr())
    torch.cuda.synchronize()
    assert int(ok.cpu()[0]) == 1
    Ln = L.cpu().numpy()
    assert np.max(np.abs(Ln - np.linalg.cholesky(A))) <= 1e-10 * np.max(np.abs(A))
    xr = np.linalg.solve(A, b)
    assert np.max(np.abs(x.cpu().numpy() - xr)) <= 1e-9 * max(1.0, np.max(np.abs(xr)))


def test_plugin_linearizer_and_reference_style_state(pkg):
    """The reference's plug-in point (mpc.py:23, :82-87): mpc_step accepts any
    callable returning LinearizedDynamics-like NumPy blocks and a NumPy
    MpcState-like object; stages 2-4 still run on the GPU."""
    from types import SimpleNamespace

    from oracle import ref_port as O

    cs = pipeline_case("p4_interior")
    N, M = cs.spec.horizon, cs.topo.node_count
    E = len(cs.topo.edges)
    rng = np.random.default_rng(0)
    A = np.eye(6) + 0.01 * rng.standard_normal((6, 6))
    Bm = 0.01 * rng.standard_normal((6, 6))

    def linearizer(states, inputs):
        K = inputs.shape[0]
        return SimpleNamespace(topology=cs.topo, horizon=K, a_self=np.tile(A, (K, M, 1, 1)),
                               a_nbr=np.full((K, E, 6, 6), 1e-3), b=np.tile(Bm, (K, M, 1, 1)),
                               c=np.zeros((K, M, 6)), n_state=6, n_u=6)

    state = SimpleNamespace(lin_states=np.tile(cs.x0, (N + 1, 1, 1)), lin_inputs=np.zeros((N, 6)),
                            step_count=0, last_applied=None, filtered_input=None)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    u, st1 = pkg.mpc_step(linearizer, cs.topo, cs.spec, pkg.SystemState(cs.x0), state, cfg)
    lin = linearizer(state.lin_states[:N], state.lin_inputs)
    gu, gx = O.condense_gammas(lin, cs.x0)
    qp = O.condense_ocp(cs.spec, lin, cs.x0, gammas=(gu, gx))
    H, g, C, d, n0 = O.expand_soft_constraints(qp)
    sol = O.solve_qp(H, g, C, d, warm_start=np.zeros(H.shape[0]))
    assert st1.last_status.value == sol.status
    assert np.max(np.abs(u.u - sol.u[:6])) <= 1e-4 * max(1.0, np.max(np.abs(sol.u)))


# ---------------------------------------------------------------------------
# mpc_step branches (reference mpc.py:129-200): SQP loop, damping, input
# filter, cold start, both fallback policies (forced primal-infeasible QP)
# ---------------------------------------------------------------------------
BRANCH_CFG = {"sqp2": dict(sqp_iterations=2), "damp": dict(sqp_damping=0.5),
              "sqp2damp": dict(sqp_iterations=2, sqp_damping=0.5),
              "filter": dict(input_filter_tau=0.05), "fbhold": {},
              "fbzero": dict(fallback="zero-input"), "fbfirst": {}, "coldstart": dict(warm_start=False)}
BRANCH_SPECS = {"fbhold": ("spec", "bad", "spec"), "fbzero": ("spec", "bad", "spec"),
                "fbfirst": ("bad", "spec")}


@pytest.mark.parametrize("case", sorted(BRANCH_CFG))
def test_mpc_step_branches_match_reference(pkg, case):
    bc = mpc_branch_cases()
    steps = bc.cases[case]
    N = bc.spec.horizon
    cfg = pkg.MpcConfig(horizon=N, dt=0.01, **BRANCH_CFG[case])
    names = BRANCH_SPECS.get(case, ("spec",) * len(steps))
    st = pkg.mpc_init(pkg.SystemState(bc.x_seq[0]), cfg, 6)
    prev_applied = None
    for t, ref in enumerate(steps):
        u, st = pkg.mpc_step(bc.model, bc.topo, getattr(bc, names[t]), pkg.SystemState(bc.x_seq[t]),
                             st, cfg)
        info = (case, t)
        assert st.last_status.value == STATUS[int(ref["meta"][0])], info
        assert abs(st.last_iterations - int(ref["meta"][1])) <= cfg.sqp_iterations, info
        scale = max(1.0, float(np.max(np.abs(ref["u"]))))
        assert float(np.max(np.abs(u.u - ref["u"]))) / scale <= TOL, info
        assert float(np.max(np.abs(st.last_applied - ref["last_applied"]))) / scale <= TOL, info
        assert rel(st.lin_states, ref["lin_states"]) <= TOL, info
        assert float(np.max(np.abs(st.lin_inputs - ref["lin_inputs"]))) / scale <= TOL, info
        assert rel(st.planned_states, ref["planned_states"]) <= TOL, info
        assert float(np.max(np.abs(st.planned_inputs - ref["planned_inputs"]))) / scale <= TOL, info
        if ref["filtered"].size:
            assert float(np.max(np.abs(st.filtered_input - ref["filtered"]))) / scale <= TOL, info
        if STATUS[int(ref["meta"][0])] == "primal_infeasible":
            # the fallback input is exact: this controller's own held input
            # (hold-previous-input after a solved step) or zeros
            expect = prev_applied if (cfg.fallback == "hold-previous-input"
                                      and prev_applied is not None) else np.zeros(6)
            assert np.array_equal(u.u, expect), info
        prev_applied = np.array(st.last_applied)


# ---------------------------------------------------------------------------
# known-answer tests of the reference suite on the GPU path
# ---------------------------------------------------------------------------

def test_relu_subgradient_zero_at_kink(pkg):
    """Pre-activations exactly 0 take derivative 0 (mlp.py:143 strict > 0,
    reference tests/test_mlp.py:84-90): zero biases, zero normalisation mean
    and the all-zero linearisation point make every pre-activation of psi and
    phi exactly 0, so every Jacobian vanishes and A = [[I, dt I],[0, I]],
    A_nbr = 0, B = 0 exactly, for every linearisation kernel."""
    rng = np.random.default_rng(8)
    topo = pkg.chain_topology(5)
    model = pkg.init_model(3, 6, 0.02, rng, n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64))
    N = 3
    expect = np.block([[np.eye(3), 0.02 * np.eye(3)], [np.zeros((3, 3)), np.eye(3)]])
    for mode in (1, 2, 3, 4):
        _set_lin_mode(pkg, SimpleNamespace(topo=topo, model=model), mode)
        try:
            lin = pkg.linearize_trajectory(model, topo, np.zeros((N, 5, 6)), np.zeros((N, 6)))
        finally:
            _set_lin_mode(pkg, SimpleNamespace(topo=topo, model=model), 0)
        # blocks are stored in fp32: exactly the fp32 rounding of the expectation
        e32 = expect.astype(np.float32).astype(float)
        assert np.array_equal(lin.a_self, np.broadcast_to(e32, lin.a_self.shape)), mode
        assert not np.any(lin.a_nbr) and not np.any(lin.b) and not np.any(lin.c), mode
    # just above the kink the derivative is 1 (the reference's J_pos case):
    # a point with every pre-activation > 0 must give non-zero Jacobians
    lin = pkg.linearize_trajectory(model, topo, np.full((N, 5, 6), 1e-3), np.full((N, 6), 1e-3))
    assert np.any(lin.b)


def test_linearize_zero_network_blocks(pkg):
    """All-zero weights (reference tests/test_gnn.py:157-166): A = [[I, dt I],
    [0, I]], B = 0, c = 0, A_nbr = 0 at any point."""
    from paper_2602_17601_b200.mlp import MlpParams

    rng = np.random.default_rng(2)
    m0 = pkg.init_model(2, 3, 0.04, rng, n_m=4, psi_hidden=(6,), phi_hidden=(6,))

    def zero(mlp):
        return MlpParams(list(mlp.layer_dims), [np.zeros_like(W) for W in mlp.weights],
                         [np.zeros_like(b) for b in mlp.biases])

    model = pkg.GnnModel(zero(m0.psi), zero(m0.phi), 0.04, 2, 3, 4, m0.normalization)
    topo = pkg.chain_topology(3)
    lin = pkg.linearize_trajectory(model, topo, np.ones((1, 3, 4)), np.zeros((1, 3)))
    expected = np.block([[np.eye(2), 0.04 * np.eye(2)], [np.zeros((2, 2)), np.eye(2)]])
    e32 = expected.astype(np.float32).astype(float)  # blocks are stored in fp32
    for i in range(3):
        assert np.array_equal(lin.a_self[0, i], e32)
        assert not np.any(lin.b[0, i])
        # c = f - A x - B u in fp64 from the stored fp32 blocks: fp32(dt) * x
        # leaves ~1e-9 (the reference test's own check is allclose(c, 0))
        assert np.allclose(lin.c[0, i], 0)
    assert not np.any(lin.a_nbr)


def test_single_node_ignores_edge_function(pkg):
    """A single node has no edges, so psi never enters (reference
    tests/test_gnn.py:75-84): step_array and the linearisation are bitwise
    independent of the psi weights."""
    rng = np.random.default_rng(4)
    topo = pkg.chain_topology(1)
    m1 = pkg.init_model(2, 3, 0.02, rng, n_m=4, psi_hidden=(6,), phi_hidden=(6,))
    m2 = m1.copy()
    for w in m2.psi.weights:
        w[...] = rng.standard_normal(w.shape)
    x = rng.standard_normal((2, 1, 4))
    u = rng.standard_normal((2, 3))
    f1 = pkg.step_array(m1, topo, x, u)
    f2 = pkg.step_array(m2, topo, x, u)
    assert np.array_equal(f1, f2)
    l1 = pkg.linearize_trajectory(m1, topo, x, u)
    l2 = pkg.linearize_trajectory(m2, topo, x, u)
    for k in ("a_self", "b", "c"):
        assert np.array_equal(getattr(l1, k), getattr(l2, k)), k


@pytest.mark.parametrize("n", [120, 128, 136, 160])
def test_qp_factor_block_sizes(pkg, n):
    """Dense QPs across the solver's substitution variants: 16-row blocks for
    T = ceil(n/8) <= 16 (odd and even T), 8-row blocks beyond; box rows plus
    general rows, against the oracle IPM (qpsolver.py:112-235): same status,
    iterations +-1, |du| <= 1e-6."""
    from oracle import ref_port as O

    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    H = A @ A.T / n + np.eye(n) * 0.1
    g = rng.standard_normal(n) * 3.0
    ng = 12
    Cg = rng.standard_normal((ng, n))
    C = np.vstack([np.eye(n), -np.eye(n), Cg])
    d = np.concatenate([np.full(n, 0.4), np.full(n, 0.4), np.abs(rng.standard_normal(ng)) + 0.2])
    ref = O.solve_qp(H, g, C, d)
    sol = pkg.solve_qp(pkg.QpProblem(H, g, C, d))
    info = (n, sol.status.value, ref.status, sol.iterations, ref.iterations)
    assert sol.status.value == ref.status, info
    assert abs(sol.iterations - ref.iterations) <= 1, info
    assert np.max(np.abs(sol.u - ref.u)) <= 1e-6, info


def test_qp_too_large_fails_loudly(pkg):
    """Beyond the on-chip capacity (vectors + factor tiles > shared memory)
    the solver refuses with a ConfigurationError instead of degrading."""
    from paper_2602_17601_b200.errors import ConfigurationError

    n = 200
    C = np.vstack([np.eye(n), -np.eye(n), np.ones((12, n))])
    with pytest.raises(ConfigurationError):
        pkg.solve_qp(pkg.QpProblem(np.eye(n), np.ones(n), C, np.ones(2 * n + 12)))
