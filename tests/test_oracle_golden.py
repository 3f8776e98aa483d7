"""Pin the CPU oracle (oracle/ref_port.py) against golden vectors produced by
the reference itself (oracle/make_golden.py), and pin the synthetic-workload
generator against the reference's own recipe (experiments.py:465-489).
CPU only."""

import numpy as np
import pytest

from oracle import ref_port as O
from tests.golden_io import (STATUS, load, local_condense_cases, training_cases, mpc_branch_cases, pipeline_case, qp_round2,
                             random_condense_cases, random_qps, rel, topo_from_ptr)

CASES = ["cfg1_chain10", "p3_biases_norm", "p4_interior", "mesh6x5", "mesh_p3"]

# MpcConfig of each reference branch sequence (oracle/make_golden.py round2)
BRANCH_CFG = {"sqp2": dict(sqp_iterations=2), "damp": dict(sqp_damping=0.5),
              "sqp2damp": dict(sqp_iterations=2, sqp_damping=0.5),
              "filter": dict(input_filter_tau=0.05), "fbhold": {},
              "fbzero": dict(fallback="zero-input"), "fbfirst": {}, "coldstart": dict(warm_start=False)}
BRANCH_SPECS = {"fbhold": ("spec", "bad", "spec"), "fbzero": ("spec", "bad", "spec"),
                "fbfirst": ("bad", "spec")}


@pytest.mark.parametrize("name", CASES)
def test_oracle_pipeline_matches_reference(name):
    cs = pipeline_case(name)
    d = cs.d
    lin = O.linearize_trajectory(cs.model, cs.topo, cs.states, cs.inputs)
    for k in ("a_self", "a_nbr", "b", "c"):
        assert np.max(np.abs(getattr(lin, k) - d["lin_" + k])) <= 1e-13, k
    gu, gx = O.condense_gammas(lin, cs.x0)
    assert rel(gu, d["gamma_u"]) <= 1e-13 and rel(gx, d["gamma_x"]) <= 1e-13
    qp = O.condense_ocp(cs.spec, lin, cs.x0, gammas=(gu, gx))
    assert rel(qp.h, d["qp_h"]) <= 1e-13 and rel(qp.g, d["qp_g"]) <= 1e-13
    if qp.c.size:
        assert rel(qp.c, d["qp_c"]) <= 1e-13
    assert np.array_equal(qp.soft, d["qp_soft"])
    H, g, C, dd, n0 = O.expand_soft_constraints(qp)
    assert rel(H, d["x_H"]) <= 1e-13 and rel(C, d["x_C"]) <= 1e-13
    sol = O.solve_qp(H, g, C, dd)
    assert sol.status == STATUS[int(d["sol_meta"][0])]
    assert sol.iterations == int(d["sol_meta"][1])
    assert np.max(np.abs(sol.u - d["sol_u"])) <= 1e-8
    rec = O.reconstruct_states(gu, gx, sol.u[:n0])
    assert rel(rec, d["recon"]) <= 1e-10
    out = O.mpc_step(cs.model, cs.topo, cs.spec, cs.x0, np.tile(cs.x0, (cs.spec.horizon + 1, 1, 1)),
                     np.zeros((cs.spec.horizon, cs.spec.n_u)), cs.spec.horizon)
    assert out["status"] == STATUS[int(d["mpc_meta"][0])]
    assert np.max(np.abs(out["u_applied"] - d["mpc_u"])) <= 1e-8
    assert rel(out["lin_states"], d["mpc_lin_states"]) <= 1e-10
    out2 = O.mpc_step(cs.model, cs.topo, cs.spec, cs.x0, out["lin_states"], out["lin_inputs"],
                      cs.spec.horizon)
    assert np.max(np.abs(out2["u_applied"] - d["mpc2_u"])) <= 1e-8


def test_oracle_random_condense_instances():
    for t, cs in enumerate(random_condense_cases()):
        gu, gx = O.condense_gammas(cs.lin, cs.x0)
        assert rel(gu, cs.gamma_u) <= 1e-13, t
        assert rel(gx, cs.gamma_x) <= 1e-13, t
        qp = O.condense_ocp(cs.spec, cs.lin, cs.x0)
        assert rel(qp.h, cs.qp["h"]) <= 1e-13, t
        assert rel(qp.g, cs.qp["g"]) <= 1e-13, t
        assert qp.c.shape == cs.qp["c"].shape
        assert np.array_equal(qp.soft, cs.qp["soft"])


def test_oracle_random_qps():
    for t, q in enumerate(random_qps()):
        sol = O.solve_qp(q.H, q.g, q.C, q.d)
        assert sol.status == q.status, t
        assert sol.iterations == q.iterations, t
        assert np.max(np.abs(sol.u - q.u)) <= 1e-9, t


def test_oracle_graph_tables():
    d = load("graph_tables")
    names = sorted({k.rsplit("_", 2)[0] for k in d if k.endswith("_nbr_ptr")})
    assert names
    for name in names:
        topo = topo_from_ptr(d[name + "_nbr_ptr"], d[name + "_nbr_list"], d[name + "_bound"])
        dst, src, gather = O.edge_lists(topo)
        nbr_idx, slots = O.slot_tables(topo)
        assert np.array_equal(dst, d[name + "_dst"]) and np.array_equal(src, d[name + "_src"])
        assert np.array_equal(gather, d[name + "_gather"])
        assert np.array_equal(nbr_idx, d[name + "_nbr_idx"])
        assert np.array_equal(slots, d[name + "_edge_slot"])


def test_workload_generator_matches_reference_recipe():
    """workloads.scaling_problem reproduces _scaling_problem bit for bit."""
    from paper_2602_17601_b200 import workloads

    cs = pipeline_case("cfg1_chain10")
    topo, model, states, inputs, spec = workloads.scaling_problem(10, 10, 0.01, 0)
    assert np.array_equal(states, cs.states) and np.array_equal(inputs, cs.inputs)
    for a, b in zip(model.psi.weights + model.phi.weights,
                    cs.model.psi.weights + cs.model.phi.weights):
        assert np.array_equal(a, b)
    assert np.array_equal(spec.q, cs.spec.q) and np.array_equal(spec.x_ref, cs.spec.x_ref)
    assert np.array_equal(spec.r, cs.spec.r)
    assert [(s.node, s.stage, s.soft) for s in spec.state_constraints] == \
        [(s.node, s.stage, s.soft) for s in cs.spec.state_constraints]
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
               for a, b in zip(spec.input_constraints, cs.spec.input_constraints))


def test_hand_known_answers():
    """Known answers from the reference tests."""
    from types import SimpleNamespace

    from paper_2602_17601_b200.graph import GraphTopology, chain_topology

    topo = GraphTopology(1, ((),), 1)
    lin = SimpleNamespace(topology=topo, horizon=2, a_self=np.full((2, 1, 1, 1), 2.0),
                          a_nbr=np.zeros((2, 0, 1, 1)), b=np.full((2, 1, 1, 1), 1.0),
                          c=np.zeros((2, 1, 1)))
    gu, gx = O.condense_gammas(lin, np.array([[1.0]]))
    assert np.allclose(gu[0].reshape(3, 2), [[0, 0], [1, 0], [2, 1]])
    assert np.allclose(gx[0].reshape(3), [1, 2, 4])
    sol = O.solve_qp(np.array([[1.0]]), np.array([-2.0]), np.array([[1.0]]), np.array([0.5]))
    assert sol.status == "optimal" and abs(sol.u[0] - 0.5) <= 1e-7 and abs(sol.duals[0] - 1) <= 1e-6
    t3 = chain_topology(3)
    assert t3.edges == [(0, 1), (1, 0), (1, 2), (2, 1)]
    assert t3.closed_neighbors(1) == (1, 0, 2)


def _cfg2():
    from tests.golden_io import model_from

    d = load("cfg2_closed_loop")
    model = model_from(d, "m_")
    from paper_2602_17601_b200.graph import chain_topology

    return d, model, chain_topology(d["x0"].shape[0])


def test_oracle_plant_matches_reference():
    """trunk.py step_state_array (one controller period, 10 substeps)."""
    d, _, _ = _cfg2()
    P = O.trunk_params(d["x0"].shape[0])
    out = O.trunk_step(P, d["plant_in"], d["plant_u"])
    assert np.max(np.abs(out - d["plant_out"])) <= 1e-12


def test_oracle_closed_loop_matches_reference():
    """run_closed_loop with the reference's tracking provider and plant (cfg2
    stack at M=10, N=10, 6 steps)."""
    d, model, topo = _cfg2()
    M = d["x0"].shape[0]
    P = O.trunk_params(M)
    specs = O.tracking_specs(topo, 10, 0.01, d["x0"], O.circle_ref(0.04, 8.0, d["center"]), 6, 8.0)
    states, inputs, statuses, iters = O.closed_loop(model, topo, P, specs, d["x0"], 6, 10)
    assert [s for s in statuses] == [str(s) for s in d["statuses"]]
    assert np.array_equal(iters, d["iterations"])
    assert np.max(np.abs(inputs - d["inputs"])) <= 1e-7
    assert np.max(np.abs(states - d["states"])) <= 1e-9


@pytest.mark.parametrize("case", sorted(BRANCH_CFG))
def test_oracle_mpc_branches_match_reference(case):
    """The oracle's mpc_step under the SQP loop, damping, input filter,
    cold start and both fallback policies equals the reference's
    (mpc.py:129-200)."""
    bc = mpc_branch_cases()
    steps = bc.cases[case]
    kw = dict(BRANCH_CFG[case])
    N = bc.spec.horizon
    tau = kw.pop("input_filter_tau", None)
    warm = kw.pop("warm_start", True)
    names = BRANCH_SPECS.get(case, ("spec",) * len(steps))
    ls, li = np.tile(bc.x_seq[0], (N + 1, 1, 1)), np.zeros((N, 6))
    last, filt = None, None
    for t, ref in enumerate(steps):
        spec = getattr(bc, names[t])
        out = O.mpc_step(bc.model, bc.topo, spec, bc.x_seq[t], ls, li, N, warm_start=warm,
                         last_applied=last, input_filter_tau=tau, filtered_input=filt, dt=0.01, **kw)
        assert out["status"] == STATUS[int(ref["meta"][0])], (case, t)
        assert out["iterations"] == int(ref["meta"][1]), (case, t)
        assert np.max(np.abs(out["u_applied"] - ref["u"])) <= 1e-8, (case, t)
        assert np.max(np.abs(out["lin_states"] - ref["lin_states"])) <= 1e-9, (case, t)
        assert np.max(np.abs(out["lin_inputs"] - ref["lin_inputs"])) <= 1e-8, (case, t)
        assert np.max(np.abs(out["planned_states"] - ref["planned_states"])) <= 1e-9, (case, t)
        ls, li, last, filt = out["lin_states"], out["lin_inputs"], out["u_applied"], out["filtered_input"]


def test_oracle_qp_round2_fixtures():
    """Best iterate at the iteration cap (tests/test_qpsolver.py:127-134),
    same-shape batches, the infeasible KAT (:119-124)."""
    q2 = qp_round2()
    for t, q in enumerate(q2.cap + q2.batch):
        sol = O.solve_qp(q.H, q.g, q.C, q.d, max_iterations=q.cap)
        assert sol.status == q.status and sol.iterations == q.iterations, t
        assert np.max(np.abs(sol.u - q.u)) <= 1e-9, t
    sol = O.solve_qp(np.array([[1.0]]), np.zeros(1), np.array([[1.0], [-1.0]]), np.array([-1.0, -2.0]))
    assert sol.status == q2.infeas_status == "primal_infeasible"
    assert sol.iterations == q2.infeas_iterations
    assert np.array_equal(sol.u, q2.infeas_u)


def test_oracle_local_condensing_matches_reference():
    """condense_local / local_hessian_gradient / assemble_qp restated
    (condensing.py:231-360) against the reference's own outputs."""
    for t, cs in enumerate(local_condense_cases()):
        locs = O.condense_local(cs.spec, cs.lin, cs.x0)
        assert np.max(np.abs(np.stack([lc.h for lc in locs]) - cs.h)) <= 1e-12, t
        assert np.max(np.abs(np.stack([lc.g for lc in locs]) - cs.g)) <= 1e-12, t
        qa = O.assemble_qp(cs.spec, locs)
        for k in ("h", "g", "c", "d"):
            assert np.max(np.abs(getattr(qa, k) - cs.qa[k]), initial=0.0) <= 1e-12, (t, k)
        assert np.array_equal(qa.soft, cs.qa["soft"])
        q_lin, _ = O.standard_form(cs.spec)
        h0, g0 = O.local_hessian_gradient(locs[0].gamma_u, locs[0].gamma_x, cs.spec.q[0], q_lin[0])
        assert np.max(np.abs(h0 - cs.lhg_h)) <= 1e-12 and np.max(np.abs(g0 - cs.lhg_g)) <= 1e-12


def test_oracle_loss_gradients_match_reference():
    """training.py:99-150 restated, against the reference's own values."""
    for cs in training_cases():
        L, grads = O.loss_gradients(cs.model, cs.topo, cs.X, cs.U, cs.Xn, cs.W, cs.lam)
        flat = np.concatenate([g.ravel() for g in grads])
        assert abs(L - cs.loss) <= 1e-12 * max(1.0, abs(cs.loss)), cs.name
        assert np.max(np.abs(flat - cs.grads)) <= 1e-12 * max(1.0, np.max(np.abs(cs.grads))), cs.name
