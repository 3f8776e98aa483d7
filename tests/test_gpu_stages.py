"""GPU parity of every hot-path stage against the reference's golden vectors
and the CPU oracle (oracle/ref_port.py).

Tolerances (fp32 stages vs the fp64 reference):
  index tables                         bit-exact
  a_self, a_nbr, b, Gamma, H, g, C, d  rel = max|x - ref| / max|ref| <= 1e-4
  c                                     max|dc| / max|x_hat| <= 1e-4
  QP on identical fp64 data (K-QP)     |du| <= 1e-6 (reference tests' own bound)
  u* through the whole pipeline        max|du| / max(1, max|u|) <= 1e-4
"""

import numpy as np
import pytest

from tests.golden_io import STATUS, pipeline_case, random_condense_cases, random_qps, rel

pytestmark = pytest.mark.gpu

TOL = 1e-4
CASES = ["cfg1_chain10", "p3_biases_norm", "p4_interior"]


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
    qs = [q for q in random_qps() if q.H.shape[0] == 3 and q.C.shape[0] == 4]
    if len(qs) < 2:
        pytest.skip("fixture has too few same-shape QPs")
    sols = pkg.solve_qp_batched(np.stack([q.H for q in qs]), np.stack([q.g for q in qs]),
                                np.stack([q.C for q in qs]), np.stack([q.d for q in qs]))
    for q, s in zip(qs, sols):
        assert np.max(np.abs(s.u - q.u)) <= 1e-6


def test_qp_known_answers(pkg):
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.array([-2.0]), np.zeros((0, 1)), np.zeros(0)))
    assert s.status == pkg.QpStatus.OPTIMAL and abs(s.u[0] - 1.0) <= 1e-12
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.array([-2.0]), np.array([[1.0]]), np.array([0.5])))
    assert s.status == pkg.QpStatus.OPTIMAL
    assert abs(s.u[0] - 0.5) <= 1e-7 and abs(s.duals[0] - 1.0) <= 1e-6
    s = pkg.solve_qp(pkg.QpProblem(np.array([[1.0]]), np.zeros(1), np.array([[1.0], [-1.0]]),
                                   np.array([-1.0, -2.0])))
    assert s.status in (pkg.QpStatus.PRIMAL_INFEASIBLE, pkg.QpStatus.MAX_ITERATIONS)
    assert s.primal_infeas > 1e-3


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
