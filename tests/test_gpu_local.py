"""Per-node condensing on the GPU: local_hessian_gradient,
condense_local, assemble_qp (reference condensing.py:231-360) against the
reference's own outputs (tests/golden/local_condense.npz) and the
reference test-suite's known answers (tests/test_condensing.py:196-278).

Tolerances: fp32 Gamma on the device, fp64 products and sums; every array
max|d| / max|ref| <= 1e-4 like the other fp32 stages (observed ~1e-7); the
node contributions are exactly symmetric by construction (reference bound
1e-14, tests/test_condensing.py:229-235).
"""

import numpy as np
import pytest

from tests.golden_io import local_condense_cases, pipeline_case, rel

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_17601_b200 as p

    return p


def _scalar_lin(pkg, a, b, c, n_stages, x0):
    topo = pkg.GraphTopology(1, ((),), 1)
    lin = pkg.LinearizedDynamics(topo, n_stages, np.full((n_stages, 1, 1, 1), float(a)),
                                 np.zeros((n_stages, 0, 1, 1)), np.full((n_stages, 1, 1, 1), float(b)),
                                 np.full((n_stages, 1, 1), float(c)))
    return lin, np.array([[float(x0)]])


def test_local_hessian_gradient_cases(pkg):
    """tests/test_condensing.py:196-218: a cost-free node, and the scalar
    N=1 case H=1, g=2 whose optimum with R=0.5 is u* = -2/3."""
    rng = np.random.default_rng(3)
    gu = rng.standard_normal((3, 2, 4))
    gx = rng.standard_normal((3, 2))
    ql = rng.standard_normal((3, 2))
    h, g = pkg.local_hessian_gradient(gu, gx, np.zeros((3, 2, 2)), ql)
    assert np.allclose(h, 0)
    assert np.allclose(g, np.einsum("kab,ka->b", gu, ql), rtol=1e-6, atol=1e-6)
    lin, x0 = _scalar_lin(pkg, 1.0, 1.0, 0.0, 1, 1.0)
    gu, gx = pkg.condense_gammas(lin, x0)
    h, g = pkg.local_hessian_gradient(gu[0], gx[0], np.ones((2, 1, 1)), np.zeros((2, 1)))
    assert h[0, 0] == pytest.approx(1.0)
    assert g[0] == pytest.approx(2.0)
    assert -g[0] / (2 * (h[0, 0] + 0.5)) == pytest.approx(-2.0 / 3.0)


def test_local_condensing_matches_reference(pkg):
    for t, cs in enumerate(local_condense_cases()):
        locs = pkg.condense_local(cs.spec, cs.lin, cs.x0)
        H = np.stack([lc.h for lc in locs])
        G = np.stack([lc.g for lc in locs])
        assert rel(H, cs.h) <= TOL, t
        assert rel(G, cs.g) <= TOL, t
        for lc in locs:  # symmetric per node (reference: <= 1e-14)
            assert np.array_equal(lc.h, lc.h.T)
        assert [lc.c_rows.shape[0] for lc in locs] == cs.rows.tolist(), t
        if cs.c_rows.size:
            assert rel(np.concatenate([lc.c_rows for lc in locs]), cs.c_rows) <= TOL, t
        qa = pkg.assemble_qp(cs.spec, locs)
        for k in ("h", "g", "c", "d"):
            if cs.qa[k].size:
                assert rel(getattr(qa, k), cs.qa[k]) <= TOL, (t, k)
        assert np.array_equal(qa.soft, cs.qa["soft"])
        assert np.array_equal(qa.h, qa.h.T)
        # single-node API on node 0
        cost = pkg.cost_to_standard_form(cs.spec)
        h0, g0 = pkg.local_hessian_gradient(locs[0].gamma_u, locs[0].gamma_x, cost.q_blocks[0],
                                            cost.q_lin[0])
        assert rel(h0, cs.lhg_h) <= TOL and rel(g0, cs.lhg_g) <= TOL, t


@pytest.mark.parametrize("name", ["cfg1_chain10", "p3_biases_norm", "mesh6x5", "mesh_p3"])
def test_local_equals_fused(pkg, name):
    """fused = local (reference tests/test_condensing.py:264-278): the
    assembled per-node QP equals condense_ocp on the same instance, and both
    equal the reference's condensed QP."""
    cs = pipeline_case(name)
    lin = pkg.linearize_trajectory(cs.model, cs.topo, cs.states, cs.inputs)
    qf = pkg.condense_ocp(cs.spec, lin, cs.x0)
    qa = pkg.assemble_qp(cs.spec, pkg.condense_local(cs.spec, lin, cs.x0))
    for k in ("h", "g", "c", "d"):
        assert rel(getattr(qa, k), getattr(qf, k)) <= TOL, k
        assert rel(getattr(qa, k), cs.d["qp_" + k]) <= TOL, k
    assert np.array_equal(qa.soft, qf.soft)


def test_assemble_input_only_constraints(pkg):
    """tests/test_condensing.py:238-251 (exact rows)."""
    lin, x0 = _scalar_lin(pkg, 1.0, 1.0, 0.0, 2, 0.5)
    cu = [(np.array([[1.0], [-1.0]]), np.array([2.0, 0.0]))] * 2
    spec = pkg.OcpSpec(lin.topology, 2, np.zeros((1, 3, 1, 1)), np.zeros((1, 3, 1)),
                       np.tile(np.eye(1), (2, 1, 1)), np.zeros((2, 1)), cu, [])
    qp = pkg.assemble_qp(spec, pkg.condense_local(spec, lin, x0))
    expect_c = np.zeros((4, 2))
    expect_c[0, 0], expect_c[1, 0], expect_c[2, 1], expect_c[3, 1] = 1.0, -1.0, 1.0, -1.0
    assert np.array_equal(qp.c, expect_c)
    assert np.array_equal(qp.d, [2.0, 0.0, 2.0, 0.0])


def test_assemble_two_identical_nodes(pkg):
    """tests/test_condensing.py:254-261: a decoupled pair sums to twice one
    node's Hessian plus R-bar."""
    topo = pkg.GraphTopology(2, ((), ()), 1)
    N = 2
    lin = pkg.LinearizedDynamics(topo, N, np.full((N, 2, 1, 1), 0.7), np.zeros((N, 0, 1, 1)),
                                 np.full((N, 2, 1, 1), 1.0), np.zeros((N, 2, 1)))
    spec = pkg.OcpSpec(topo, N, np.full((2, N + 1, 1, 1), 1.3), np.zeros((2, N + 1, 1)),
                       np.tile(np.eye(1) * 0.2, (N, 1, 1)), np.zeros((N, 1)))
    locs = pkg.condense_local(spec, lin, np.array([[0.5], [0.5]]))
    qp = pkg.assemble_qp(spec, locs)
    assert np.allclose(qp.h, 2 * locs[0].h + np.eye(2) * 0.2, rtol=1e-6)
