"""Generate golden fixtures from the REFERENCE implementation (test infrastructure).

Runs only in the build container, where the read-only reference package is
importable from /root/reference/pkg/src.  Writes small compressed fixtures to
tests/golden/ that pin (a) the oracle port (oracle/ref_port.py) and (b) the
GPU path, on the GPU box where the reference does not exist.

    python oracle/make_golden.py

Every fixture is produced by calling the reference's own public functions;
nothing in here reimplements the algorithm.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GNNMPC_REF", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import gnnmpc.condensing as rc
    import gnnmpc.experiments as rex
    import gnnmpc.gnn as rg
    import gnnmpc.graph as rgr
    import gnnmpc.mlp as rmlp
    import gnnmpc.mpc as rm
    import gnnmpc.qpsolver as rq
    return rc, rex, rg, rgr, rmlp, rm, rq


def cfg2_closed_loop():
    """Closed-loop tracking with the reference's own plant, provider and
    run_closed_loop (cfg2 stack, reduced: M=10 nodes, N=10, 6 steps after a
    0.5 s settle; circle r=0.04 m, period 8 s around the settled tip), plus
    single plant steps at random states / inputs."""
    sys.path.insert(0, str(REF))
    import gnnmpc.experiments as rex
    import gnnmpc.gnn as rg
    import gnnmpc.graph as rgr
    import gnnmpc.mpc as rm
    import gnnmpc.references as rr
    import gnnmpc.trunk as rt

    out = {}
    M, N, steps = 10, 10, 6
    pc = rt.ChainConfig(node_count=M)
    x0 = rt.settle(pc, 0.5)
    topo = rgr.chain_topology(M)
    model = rg.init_model(3, 6, 0.01, np.random.default_rng(3), n_m=16, psi_hidden=(32, 32),
                          phi_hidden=(64, 64), out_scale=0.05)
    cfg = rm.MpcConfig(horizon=N, dt=0.01)
    center = x0.array[-1, :3].copy()
    ref = rr.circle_reference(0.04, 8.0, center)
    prov = rex.tracking_spec_provider(topo, cfg, x0, ref, rex.TrackingWeights(), pc.n_u, pc.u_max)
    log = rm.run_closed_loop(rex.make_plant_step(pc), model, topo, prov, x0, steps, cfg)
    _model_arrays("m_", model, out)
    out["x0"] = x0.array
    out["center"] = center
    out["states"] = log.states
    out["inputs"] = log.inputs
    out["iterations"] = log.iterations
    out["statuses"] = np.array([s.value for s in log.statuses])
    rng = np.random.default_rng(7)
    arr = x0.array + 0.01 * rng.standard_normal((M, 6))
    u = rng.uniform(-1.0, 9.0, 6)
    out["plant_in"] = arr
    out["plant_u"] = u
    out["plant_out"] = rt.step_state_array(pc, arr, u)
    np.savez_compressed(OUT / "cfg2_closed_loop.npz", **out)


def obstacle_provider():
    """The reference's obstacle_spec_provider (experiments.py:186-238) on a
    settled M=12 chain, N=10, evaluated at several times with no state and
    with predicted trajectories pushed towards the sphere: the OCP arrays and
    every emitted soft half-space row (node, stage, row, bound, rho)."""
    sys.path.insert(0, str(REF))
    import gnnmpc.experiments as rex
    import gnnmpc.graph as rgr
    import gnnmpc.mpc as rm
    import gnnmpc.trunk as rt

    out = {}
    M, N = 12, 10
    pc = rt.ChainConfig(node_count=M)
    x0 = rt.settle(pc, 0.5)
    topo = rgr.chain_topology(M)
    cfg = rm.MpcConfig(horizon=N, dt=0.01)
    tip = x0.array[-1, :3].copy()
    mid = 0.5 * (x0.array[-1, :3] + x0.array[-2, :3])
    scen = rex.ObstacleScenario(target_point=mid + np.array([0.05, 0.0, 0.0]),
                                approach_from=np.array([1.0, 0.0, 0.0]), constrained_nodes=(M - 1, M - 2, 5),
                                start_distance=0.3, approach_time=2.0, hold_time=1.0, retreat_time=2.0,
                                start_delay=0.2)
    prov = rex.obstacle_spec_provider(topo, cfg, x0, scen, rex.TrackingWeights(), pc.n_u, pc.u_max)
    rng = np.random.default_rng(11)
    out["x0"] = x0.array
    out["tip"] = tip
    cases = []
    for t in (0, 50, 150, 230, 300, 420):
        for with_state in (False, True):
            st = None
            if with_state:
                pred = np.repeat(x0.array[None], N + 1, axis=0) + 0.01 * rng.standard_normal((N + 1, M, 6))
                pred[:, :, 0] += np.linspace(0.0, 0.03, N + 1)[:, None]
                st = rm.MpcState(lin_states=pred, lin_inputs=np.zeros((N, pc.n_u)))
                out[f"pred_{t}"] = pred
            spec = prov(t, st)
            key = f"{t}_{int(with_state)}"
            cases.append(key)
            out[f"nodes_{key}"] = np.array([c.node for c in spec.state_constraints], dtype=np.int64)
            out[f"stages_{key}"] = np.array([c.stage for c in spec.state_constraints], dtype=np.int64)
            out[f"rows_{key}"] = np.array([c.c for c in spec.state_constraints]).reshape(-1, 6)
            out[f"bounds_{key}"] = np.array([c.d for c in spec.state_constraints]).reshape(-1)
            out[f"soft_{key}"] = np.array([c.soft for c in spec.state_constraints], dtype=bool)
            out[f"rho_{key}"] = np.array([[c.rho1, c.rho2] for c in spec.state_constraints]).reshape(-1, 2)
            out["q"], out["x_ref"], out["r"], out["u_ref"] = spec.q, spec.x_ref, spec.r, spec.u_ref
    out["cases"] = np.array(cases)
    out["centers"] = scen.center(np.arange(0, 6.0, 0.01))
    np.savez_compressed(OUT / "obstacle_provider.npz", **out)


def _model_arrays(prefix, model, out):
    for name, mlp in (("psi", model.psi), ("phi", model.phi)):
        out[f"{prefix}{name}_dims"] = np.asarray(mlp.layer_dims)
        for l, (W, b) in enumerate(zip(mlp.weights, mlp.biases)):
            out[f"{prefix}{name}_W{l}"] = W
            out[f"{prefix}{name}_b{l}"] = b
    n = model.normalization
    out[f"{prefix}norm"] = np.concatenate([n.state_mean, n.state_scale, n.input_mean, n.input_scale])
    out[f"{prefix}meta"] = np.array([model.dt, model.n_p, model.n_u, model.n_m])


def _spec_arrays(prefix, spec, out):
    out[f"{prefix}q"] = spec.q
    out[f"{prefix}x_ref"] = spec.x_ref
    out[f"{prefix}r"] = spec.r
    out[f"{prefix}u_ref"] = spec.u_ref
    if spec.input_constraints is not None:
        out[f"{prefix}icons_C"] = np.stack([C for C, _ in spec.input_constraints])
        out[f"{prefix}icons_d"] = np.stack([d for _, d in spec.input_constraints])
    sc = spec.state_constraints
    out[f"{prefix}scons_meta"] = np.array([[s.node, s.stage, int(s.soft), s.rho1, s.rho2, s.c.shape[0]]
                                           for s in sc], dtype=float).reshape(-1, 6)
    out[f"{prefix}scons_c"] = (np.concatenate([s.c for s in sc]) if sc
                               else np.zeros((0, spec.q.shape[-1])))
    out[f"{prefix}scons_d"] = np.concatenate([s.d for s in sc]) if sc else np.zeros(0)


def _pipeline(prefix, model, topo, spec, states, inputs, x0, out, rc, rg, rq, rm, rgr):
    lin = rg.linearize_trajectory(model, topo, states, inputs)
    for k in ("a_self", "a_nbr", "b", "c"):
        out[f"{prefix}lin_{k}"] = getattr(lin, k)
    gu, gx = rc.condense_gammas(lin, x0)
    out[f"{prefix}gamma_u"] = gu
    out[f"{prefix}gamma_x"] = gx
    qp = rc.condense_ocp(spec, lin, x0, gammas=(gu, gx))
    for k in ("h", "g", "c", "d", "soft", "rho1", "rho2"):
        out[f"{prefix}qp_{k}"] = getattr(qp, k)
    H, g, C, d, n0 = rc.expand_soft_constraints(qp)
    out[f"{prefix}x_H"], out[f"{prefix}x_g"], out[f"{prefix}x_C"], out[f"{prefix}x_d"] = H, g, C, d
    sol = rq.solve_qp(rq.QpProblem(H, g, C, d))
    out[f"{prefix}sol_u"] = sol.u
    out[f"{prefix}sol_duals"] = sol.duals
    out[f"{prefix}sol_meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                          "numerical_failure"].index(sol.status.value),
                                         sol.iterations, sol.stationarity, sol.primal_infeas,
                                         sol.complementarity])
    out[f"{prefix}recon"] = rc.reconstruct_states(gu, gx, sol.u[:n0])
    cfg = rm.MpcConfig(horizon=spec.horizon, dt=model.dt)
    xs = rgr.SystemState(x0)
    st = rm.mpc_init(xs, cfg, spec.r.shape[-1])
    u1, st1 = rm.mpc_step(model, topo, spec, xs, st, cfg)
    out[f"{prefix}mpc_u"] = u1.u
    out[f"{prefix}mpc_lin_states"] = st1.lin_states
    out[f"{prefix}mpc_lin_inputs"] = st1.lin_inputs
    out[f"{prefix}mpc_planned_states"] = st1.planned_states
    out[f"{prefix}mpc_meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                          "numerical_failure"].index(st1.last_status.value),
                                         st1.last_iterations])
    # second step from the shifted state (warm start path)
    u2, st2 = rm.mpc_step(model, topo, spec, xs, st1, cfg)
    out[f"{prefix}mpc2_u"] = u2.u
    out[f"{prefix}mpc2_lin_states"] = st2.lin_states
    out[f"{prefix}mpc2_meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                           "numerical_failure"].index(st2.last_status.value),
                                          st2.last_iterations])


def random_instance(rng, rc, rg, rgr, max_m=8, max_nx=4, max_nu=3, max_n=10, with_constraints=True):
    """Same generator as the reference test-suite's random_instance
    (tests/test_condensing.py:40-80), so fixtures cover its case family."""
    M = int(rng.integers(1, max_m + 1))
    nx = int(rng.integers(1, max_nx + 1))
    nu = int(rng.integers(1, max_nu + 1))
    N = int(rng.integers(1, max_n + 1))
    nbrs = []
    for i in range(M):
        others = [j for j in range(M) if j != i]
        k = int(rng.integers(0, min(2, len(others)) + 1))
        pick = sorted(rng.choice(others, size=k, replace=False).tolist()) if k else []
        nbrs.append(tuple(int(v) for v in pick))
    topo = rgr.GraphTopology(M, tuple(nbrs), 2)
    E = len(topo.edges)
    scale = 0.9 / max(1, nx)
    lin = rg.LinearizedDynamics(topo, N, a_self=rng.standard_normal((N, M, nx, nx)) * scale,
                                a_nbr=rng.standard_normal((N, E, nx, nx)) * scale,
                                b=rng.standard_normal((N, M, nx, nu)),
                                c=rng.standard_normal((N, M, nx)))
    q = rng.standard_normal((M, N + 1, nx, nx))
    q = np.einsum("mkab,mkcb->mkac", q, q) * 0.3
    r = rng.standard_normal((N, nu, nu))
    r = np.einsum("kab,kcb->kac", r, r) + np.eye(nu) * 0.5
    icons, scons = None, []
    if with_constraints:
        icons = [(rng.standard_normal((2, nu)), rng.standard_normal(2)) for _ in range(N)]
        for _ in range(int(rng.integers(0, 5))):
            scons.append(rc.StateConstraint(int(rng.integers(0, M)), int(rng.integers(0, N + 1)),
                                            rng.standard_normal((1, nx)), rng.standard_normal(1)))
    spec = rc.OcpSpec(topo, N, q, rng.standard_normal((M, N + 1, nx)), r,
                      rng.standard_normal((N, nu)), icons, scons)
    return spec, lin, rng.standard_normal((M, nx))


def main():
    rc, rex, rg, rgr, rmlp, rm, rq = _ref()
    OUT.mkdir(parents=True, exist_ok=True)

    # cfg1: the reference's own benchmark recipe at chain M=10, N=10 (experiments.py:465-489)
    out = {}
    topo, model, states, inputs, spec = rex._scaling_problem(10, 10, 0.01, 0)
    out["states"], out["inputs"] = states, inputs
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    _pipeline("", model, topo, spec, states, inputs, states[0], out, rc, rg, rq, rm, rgr)
    np.savez_compressed(OUT / "cfg1_chain10.npz", **out)

    # P3: random biases + non-identity normalisation (c != 0; tests/test_gnn.py:91-93 style)
    out = {}
    rng = np.random.default_rng(77)
    topo = rgr.chain_topology(6)
    model = rg.init_model(3, 6, 0.02, rng, n_m=8, psi_hidden=(16, 12), phi_hidden=(24, 20),
                          out_scale=0.3)
    for mlp in (model.psi, model.phi):
        for b in mlp.biases:
            b[...] = 0.2 * rng.standard_normal(b.shape)
    model.normalization = rg.Normalization(0.1 * rng.standard_normal(6), rng.random(6) + 0.5,
                                           rng.standard_normal(6), rng.random(6) + 0.5)
    N = 5
    states = 0.3 * rng.standard_normal((N + 1, 6, 6))
    inputs = rng.standard_normal((N, 6))
    q = np.tile(np.diag(rng.random(6) + 0.1), (6, N + 1, 1, 1))
    spec = rc.OcpSpec(topo, N, q, 0.1 * rng.standard_normal((6, N + 1, 6)),
                      np.tile(np.eye(6) * 0.5, (N, 1, 1)), np.zeros((N, 6)),
                      [rc.stage_input_box(6, -1.0, 1.0)] * N,
                      [rc.StateConstraint(2, 3, rng.standard_normal((2, 6)), np.array([0.5, 0.2])),
                       rc.StateConstraint(5, N, np.eye(6)[:1], np.array([0.1]), soft=True,
                                          rho1=10.0, rho2=100.0)])
    out["states"], out["inputs"] = states, inputs
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    _pipeline("", model, topo, spec, states, inputs, states[0], out, rc, rg, rq, rm, rgr)
    np.savez_compressed(OUT / "p3_biases_norm.npz", **out)

    # P4: interior-solution QP (R = 1.0 I so the optimum is off the box bounds)
    out = {}
    topo, model, states, inputs, spec = rex._scaling_problem(12, 8, 0.01, 3)
    spec = rc.OcpSpec(topo, 8, spec.q, spec.x_ref, np.tile(np.eye(6) * 1.0, (8, 1, 1)),
                      spec.u_ref, spec.input_constraints, spec.state_constraints)
    out["states"], out["inputs"] = states, inputs
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    _pipeline("", model, topo, spec, states, inputs, states[0], out, rc, rg, rq, rm, rgr)
    np.savez_compressed(OUT / "p4_interior.npz", **out)

    # P2: random condensing instances from the reference test generator
    out = {}
    rng = np.random.default_rng(5)
    for t in range(12):
        spec, lin, x0 = random_instance(rng, rc, rg, rgr, with_constraints=(t % 3 != 2))
        p = f"c{t}_"
        out[p + "nbr_ptr"] = np.concatenate([[0], np.cumsum([len(n) for n in lin.topology.in_neighbors])])
        out[p + "nbr_list"] = np.array([j for ns in lin.topology.in_neighbors for j in ns], dtype=np.int64)
        for k in ("a_self", "a_nbr", "b", "c"):
            out[p + k] = getattr(lin, k)
        out[p + "x0"] = x0
        _spec_arrays(p, spec, out)
        gu, gx = rc.condense_gammas(lin, x0)
        out[p + "gamma_u"], out[p + "gamma_x"] = gu, gx
        qp = rc.condense_ocp(spec, lin, x0)
        for k in ("h", "g", "c", "d", "soft"):
            out[p + "qp_" + k] = getattr(qp, k)
    np.savez_compressed(OUT / "p2_random_condense.npz", **out)

    # QP: random feasible problems (tests/test_qpsolver.py:31-41 family) + reference solutions
    out = {}
    rng = np.random.default_rng(42)
    for t in range(40):
        n = int(rng.integers(1, 7))
        m = int(rng.integers(0, 9))
        A = rng.standard_normal((n, n))
        H = A @ A.T + np.eye(n) * (0.1 + rng.random())
        g = rng.standard_normal(n)
        uf = rng.standard_normal(n)
        C = rng.standard_normal((m, n))
        d = C @ uf + rng.random(m) + 0.05
        sol = rq.solve_qp(rq.QpProblem(H, g, C, d))
        p = f"q{t}_"
        out[p + "H"], out[p + "g"], out[p + "C"], out[p + "d"] = H, g, C, d
        out[p + "u"], out[p + "duals"] = sol.u, sol.duals
        out[p + "meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                     "numerical_failure"].index(sol.status.value), sol.iterations])
    np.savez_compressed(OUT / "qp_random.npz", **out)

    # graph index tables (gnn.py:107-126, condensing.py:158-172), bit-exact targets
    out = {}
    graphs = {"chain1": rgr.chain_topology(1), "chain3": rgr.chain_topology(3),
              "chain7": rgr.chain_topology(7),
              "iso": rgr.GraphTopology(3, ((), (), ()), 1),
              "mixed": rgr.GraphTopology(5, ((3, 1), (), (0, 4, 1), (2,), (0,)), 3)}
    rows, cols = 3, 4
    mesh = []
    for r in range(rows):
        for c in range(cols):
            ns = []
            if r > 0: ns.append((r - 1) * cols + c)
            if c > 0: ns.append(r * cols + c - 1)
            if c < cols - 1: ns.append(r * cols + c + 1)
            if r < rows - 1: ns.append((r + 1) * cols + c)
            mesh.append(tuple(ns))
    graphs["mesh3x4"] = rgr.GraphTopology(rows * cols, tuple(mesh), 4)
    for name, topo in graphs.items():
        dst, src, gather = rg._edge_index(topo)
        lin = rg.LinearizedDynamics(topo, 1, np.zeros((1, topo.node_count, 1, 1)),
                                    np.zeros((1, len(topo.edges), 1, 1)),
                                    np.zeros((1, topo.node_count, 1, 1)),
                                    np.zeros((1, topo.node_count, 1)))
        nbr_idx, _ = rc._padded_neighborhood(lin)
        # edge_slot as the reference computes it inside _padded_neighborhood
        slots = [s + 1 for ns in topo.in_neighbors for s in range(len(ns))]
        out[name + "_nbr_ptr"] = np.concatenate([[0], np.cumsum([len(n) for n in topo.in_neighbors])])
        out[name + "_nbr_list"] = np.array([j for ns in topo.in_neighbors for j in ns], dtype=np.int64)
        out[name + "_bound"] = np.array(topo.neighbor_bound)
        out[name + "_dst"], out[name + "_src"], out[name + "_gather"] = dst, src, gather
        out[name + "_nbr_idx"] = nbr_idx
        out[name + "_edge_slot"] = np.array(slots, dtype=np.int64)
        out[name + "_edges"] = np.array(topo.edges, dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(OUT / "graph_tables.npz", **out)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


def _ref_mesh(rgr, rows, cols):
    """4-neighbour grid as a reference GraphTopology (id = r*cols + c,
    in-neighbours ascending: up, left, right, down)."""
    nbrs = []
    for r in range(rows):
        for c in range(cols):
            ns = []
            if r > 0: ns.append((r - 1) * cols + c)
            if c > 0: ns.append(r * cols + c - 1)
            if c < cols - 1: ns.append(r * cols + c + 1)
            if r < rows - 1: ns.append((r + 1) * cols + c)
            nbrs.append(tuple(ns))
    return rgr.GraphTopology(rows * cols, tuple(nbrs), 4)


def _ref_mesh_problem(rc, rg, rgr, rows, cols, N, dt, seed):
    """The cfg5 recipe (workloads.mesh_problem) built from reference objects:
    _scaling_problem's draws (experiments.py:465-489) on a mesh graph."""
    rng = np.random.default_rng(seed)
    topo = _ref_mesh(rgr, rows, cols)
    M = rows * cols
    model = rg.init_model(3, 6, dt, rng, n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64),
                          out_scale=0.05)
    ids = np.arange(M)
    states = np.zeros((N, M, 6))
    states[:, :, 0] = 0.15 * (ids % cols)
    states[:, :, 2] = -0.15 * (ids // cols)
    states += 0.01 * rng.standard_normal(states.shape)
    inputs = rng.uniform(0.0, 4.0, size=(N, 6))
    q = np.zeros((M, N + 1, 6, 6))
    q[:, :] = np.diag(np.concatenate([np.full(3, 1.0), np.full(3, 0.1)]))
    x_ref = states[0][:, None, :].repeat(N + 1, axis=1)
    row = np.zeros((1, 6))
    row[0, 2] = 1.0
    scons = [rc.StateConstraint(M - 1, k, row, np.array([1.0]), soft=True) for k in range(1, N + 1)]
    spec = rc.OcpSpec(topo, N, q, x_ref, np.tile(np.eye(6) * 1e-2, (N, 1, 1)), np.zeros((N, 6)),
                      [rc.stage_input_box(6, 0.0, 8.0)] * N, scons)
    return topo, model, states, inputs, spec


def _mpc_seq(rm, rgr, model, topo, specs, x0s, cfg, prefix, out):
    """Run the reference mpc_step over a sequence of (spec, measurement) and
    record every step's outputs (mpc.py:102-200)."""
    st = rm.mpc_init(rgr.SystemState(x0s[0]), cfg, specs[0].r.shape[-1])
    for t, (spec, x) in enumerate(zip(specs, x0s)):
        u, st = rm.mpc_step(model, topo, spec, rgr.SystemState(x), st, cfg)
        p = f"{prefix}{t}_"
        out[p + "u"] = u.u
        out[p + "lin_states"] = st.lin_states
        out[p + "lin_inputs"] = st.lin_inputs
        out[p + "planned_states"] = st.planned_states
        out[p + "planned_inputs"] = st.planned_inputs
        out[p + "last_applied"] = st.last_applied
        out[p + "filtered"] = (st.filtered_input if st.filtered_input is not None
                               else np.zeros(0))
        out[p + "meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                     "numerical_failure"].index(st.last_status.value),
                                    st.last_iterations])
    out[prefix + "steps"] = np.array(len(specs))


def round2():
    """Round-2 fixtures: mesh graphs (degree 4) through the whole pipeline,
    the mpc_step branches (SQP loop, damping, input filter, both fallback
    policies), the iteration-cap best iterate and batched same-shape QPs."""
    rc, rex, rg, rgr, rmlp, rm, rq = _ref()
    OUT.mkdir(parents=True, exist_ok=True)

    # mesh 6x5 (M=30, E=98), N=6, the cfg5 recipe
    out = {}
    topo, model, states, inputs, spec = _ref_mesh_problem(rc, rg, rgr, 6, 5, 6, 0.01, 1)
    out["states"], out["inputs"] = states, inputs
    out["mesh"] = np.array([6, 5])
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    _pipeline("", model, topo, spec, states, inputs, states[0], out, rc, rg, rq, rm, rgr)
    np.savez_compressed(OUT / "mesh6x5.npz", **out)

    # P3-style mesh 4x4: random biases + normalisation (c != 0), hard and soft
    # state rows on interior (degree-4) nodes
    out = {}
    rng = np.random.default_rng(91)
    topo = _ref_mesh(rgr, 4, 4)
    M, N = 16, 5
    model = rg.init_model(3, 6, 0.02, rng, n_m=8, psi_hidden=(16, 12), phi_hidden=(24, 20),
                          out_scale=0.3)
    for mlp in (model.psi, model.phi):
        for b in mlp.biases:
            b[...] = 0.2 * rng.standard_normal(b.shape)
    model.normalization = rg.Normalization(0.1 * rng.standard_normal(6), rng.random(6) + 0.5,
                                           rng.standard_normal(6), rng.random(6) + 0.5)
    states = 0.3 * rng.standard_normal((N + 1, M, 6))
    inputs = rng.standard_normal((N, 6))
    q = np.tile(np.diag(rng.random(6) + 0.1), (M, N + 1, 1, 1))
    spec = rc.OcpSpec(topo, N, q, 0.1 * rng.standard_normal((M, N + 1, 6)),
                      np.tile(np.eye(6) * 0.5, (N, 1, 1)), np.zeros((N, 6)),
                      [rc.stage_input_box(6, -1.0, 1.0)] * N,
                      [rc.StateConstraint(5, 3, rng.standard_normal((2, 6)), np.array([0.5, 0.2])),
                       rc.StateConstraint(10, N, np.eye(6)[:1], np.array([0.1]), soft=True,
                                          rho1=10.0, rho2=100.0)])
    out["states"], out["inputs"] = states, inputs
    out["mesh"] = np.array([4, 4])
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    _pipeline("", model, topo, spec, states, inputs, states[0], out, rc, rg, rq, rm, rgr)
    np.savez_compressed(OUT / "mesh_p3.npz", **out)

    # mpc_step branches on the cfg1 recipe (chain M=10, N=10)
    out = {}
    topo, model, states, inputs, spec = rex._scaling_problem(10, 10, 0.01, 0)
    _model_arrays("", model, out)
    _spec_arrays("", spec, out)
    out["states"], out["inputs"] = states, inputs
    N = 10
    rng = np.random.default_rng(13)
    xs = [states[0] + 0.002 * rng.standard_normal(states[0].shape) for _ in range(3)]
    out["x_seq"] = np.stack(xs)
    # a spec whose QP is primal infeasible: hard rows z <= -100 and -z <= -100
    # on node 0 at stage 1 (contradictory), on top of the feasible spec
    bad_rows = np.zeros((2, 6))
    bad_rows[0, 2], bad_rows[1, 2] = 1.0, -1.0
    bad = rc.OcpSpec(topo, N, spec.q, spec.x_ref, spec.r, spec.u_ref, spec.input_constraints,
                     list(spec.state_constraints)
                     + [rc.StateConstraint(0, 1, bad_rows, np.array([-100.0, -100.0]))])
    out["bad_row_c"], out["bad_row_d"] = bad_rows, np.array([-100.0, -100.0])
    cases = {
        "sqp2": (rm.MpcConfig(horizon=N, dt=0.01, sqp_iterations=2), [spec] * 2),
        "damp": (rm.MpcConfig(horizon=N, dt=0.01, sqp_damping=0.5), [spec] * 2),
        "sqp2damp": (rm.MpcConfig(horizon=N, dt=0.01, sqp_iterations=2, sqp_damping=0.5),
                     [spec] * 2),
        "filter": (rm.MpcConfig(horizon=N, dt=0.01, input_filter_tau=0.05), [spec] * 3),
        "fbhold": (rm.MpcConfig(horizon=N, dt=0.01), [spec, bad, spec]),
        "fbzero": (rm.MpcConfig(horizon=N, dt=0.01, fallback="zero-input"), [spec, bad, spec]),
        "fbfirst": (rm.MpcConfig(horizon=N, dt=0.01), [bad, spec]),
        "coldstart": (rm.MpcConfig(horizon=N, dt=0.01, warm_start=False), [spec] * 2),
    }
    for name, (cfg, specs) in cases.items():
        _mpc_seq(rm, rgr, model, topo, specs, xs[: len(specs)], cfg, name + "_", out)
    out["cases"] = np.array(list(cases))
    np.savez_compressed(OUT / "mpc_branches.npz", **out)

    # QP: best iterate at the iteration cap (tests/test_qpsolver.py:127-134),
    # batched same-shape problems, the infeasible KAT (:119-124)
    out = {}
    rng = np.random.default_rng(21)
    k = 0
    for cap in (1, 2, 3, 5):
        for _ in range(3):
            n, m = int(rng.integers(2, 7)), int(rng.integers(1, 9))
            A = rng.standard_normal((n, n))
            H = A @ A.T + np.eye(n) * (0.1 + rng.random())
            g = rng.standard_normal(n)
            C = rng.standard_normal((m, n))
            d = C @ rng.standard_normal(n) + rng.random(m) + 0.05
            sol = rq.solve_qp(rq.QpProblem(H, g, C, d), rq.SolverSettings(max_iterations=cap))
            p = f"cap{k}_"
            out[p + "H"], out[p + "g"], out[p + "C"], out[p + "d"] = H, g, C, d
            out[p + "u"], out[p + "duals"] = sol.u, sol.duals
            out[p + "meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                         "numerical_failure"].index(sol.status.value),
                                        sol.iterations, cap])
            k += 1
    for t in range(8):
        n, m = 5, 7
        A = rng.standard_normal((n, n))
        H = A @ A.T + np.eye(n) * (0.1 + rng.random())
        g = rng.standard_normal(n)
        C = rng.standard_normal((m, n))
        d = C @ rng.standard_normal(n) + rng.random(m) + 0.05
        sol = rq.solve_qp(rq.QpProblem(H, g, C, d))
        p = f"b{t}_"
        out[p + "H"], out[p + "g"], out[p + "C"], out[p + "d"] = H, g, C, d
        out[p + "u"], out[p + "duals"] = sol.u, sol.duals
        out[p + "meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                     "numerical_failure"].index(sol.status.value), sol.iterations])
    sol = rq.solve_qp(rq.QpProblem(np.array([[1.0]]), np.zeros(1), np.array([[1.0], [-1.0]]),
                                   np.array([-1.0, -2.0])))
    out["infeas_u"] = sol.u
    out["infeas_meta"] = np.array([["optimal", "max_iterations", "primal_infeasible",
                                    "numerical_failure"].index(sol.status.value), sol.iterations,
                                   sol.primal_infeas])
    np.savez_compressed(OUT / "qp_round2.npz", **out)
    for f in ("mesh6x5", "mesh_p3", "mpc_branches", "qp_round2"):
        print(f, (OUT / f"{f}.npz").stat().st_size)


def local_condense():
    """Per-node condensing of the reference (condensing.py:231-360):
    condense_local + assemble_qp on P2-family random instances (degree <= 2,
    constraints, soft rows) and on the P3-style mesh, every node's h, g and
    rows plus the assembled QP."""
    rc, rex, rg, rgr, rmlp, rm, rq = _ref()
    out = {}
    rng = np.random.default_rng(17)
    for t in range(6):
        spec, lin, x0 = random_instance(rng, rc, rg, rgr, with_constraints=(t % 3 != 2))
        p = f"c{t}_"
        out[p + "nbr_ptr"] = np.concatenate([[0], np.cumsum([len(n) for n in lin.topology.in_neighbors])])
        out[p + "nbr_list"] = np.array([j for ns in lin.topology.in_neighbors for j in ns], dtype=np.int64)
        for k in ("a_self", "a_nbr", "b", "c"):
            out[p + k] = getattr(lin, k)
        out[p + "x0"] = x0
        _spec_arrays(p, spec, out)
        locs = rc.condense_local(spec, lin, x0)
        out[p + "h"] = np.stack([lc.h for lc in locs])
        out[p + "g"] = np.stack([lc.g for lc in locs])
        out[p + "rows"] = np.array([lc.c_rows.shape[0] for lc in locs])
        n0 = spec.horizon * spec.n_u
        out[p + "c_rows"] = np.concatenate([lc.c_rows for lc in locs]) if locs else np.zeros((0, n0))
        out[p + "d_rows"] = np.concatenate([lc.d_rows for lc in locs])
        qa = rc.assemble_qp(spec, locs)
        for k in ("h", "g", "c", "d", "soft", "rho1", "rho2"):
            out[p + "qa_" + k] = getattr(qa, k)
        # the single-node API on node 0's maps and cost
        cost = rc.cost_to_standard_form(spec)
        h0, g0 = rc.local_hessian_gradient(locs[0].gamma_u, locs[0].gamma_x, cost.q_blocks[0],
                                           cost.q_lin[0])
        out[p + "lhg_h"], out[p + "lhg_g"] = h0, g0
    np.savez_compressed(OUT / "local_condense.npz", **out)
    print("local_condense", (OUT / "local_condense.npz").stat().st_size)


def training_grads():
    """The reference's loss_gradients (training.py:99-150) on three
    instances: the reference FD test's tiny model (chain 2, l2 1e-3), the
    cfg architecture on a chain of 5, and a 3x3 mesh with random biases and
    normalisation; batch losses and every gradient."""
    sys.path.insert(0, str(REF))
    import gnnmpc.gnn as rg
    import gnnmpc.graph as rgr
    import gnnmpc.training as rt

    out = {}
    rng = np.random.default_rng(2)
    cases = []
    m = rg.init_model(1, 2, 0.05, rng, n_m=3, psi_hidden=(5,), phi_hidden=(6,))
    cases.append(("fd", rgr.chain_topology(2), m, 6, np.array([2.0, 0.5]), 1e-3))
    m = rg.init_model(3, 6, 0.01, rng, n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64), out_scale=0.05)
    cases.append(("cfg", rgr.chain_topology(5), m, 16, None, 1e-6))
    m = rg.init_model(3, 6, 0.02, rng, n_m=8, psi_hidden=(16, 12), phi_hidden=(24, 20), out_scale=0.3)
    for mlp in (m.psi, m.phi):
        for b in mlp.biases:
            b[...] = 0.2 * rng.standard_normal(b.shape)
    m.normalization = rg.Normalization(0.1 * rng.standard_normal(6), rng.random(6) + 0.5,
                                       rng.standard_normal(6), rng.random(6) + 0.5)
    cases.append(("mesh", _ref_mesh(rgr, 3, 3), m, 9, np.linspace(0.5, 2.0, 6), 0.0))
    names = []
    for name, topo, model, B, w, lam in cases:
        M, nx = topo.node_count, 2 * model.n_p
        X = rng.standard_normal((B, M, nx)) * 0.3
        U = rng.standard_normal((B, model.n_u))
        Xn = X + 0.05 * rng.standard_normal((B, M, nx))
        W = rt._weight_grid(w, M, nx)
        L, grads = rt.loss_gradients(model, topo, X, U, Xn, W, lam)
        p = name + "_"
        _model_arrays(p + "m_", model, out)
        out[p + "nbr_ptr"] = np.concatenate([[0], np.cumsum([len(n) for n in topo.in_neighbors])])
        out[p + "nbr_list"] = np.array([j for ns in topo.in_neighbors for j in ns], dtype=np.int64)
        out[p + "X"], out[p + "U"], out[p + "Xn"], out[p + "W"] = X, U, Xn, W
        out[p + "lam"] = np.array(lam)
        out[p + "loss"] = np.array(L)
        out[p + "grads"] = np.concatenate([g.ravel() for g in grads])
        names.append(name)
    out["cases"] = np.array(names)
    np.savez_compressed(OUT / "training_grads.npz", **out)
    print("training_grads", (OUT / "training_grads.npz").stat().st_size)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cfg2":
        cfg2_closed_loop()
        raise SystemExit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "round2":
        round2()
        local_condense()
        training_grads()
        raise SystemExit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "obstacle":
        obstacle_provider()
        raise SystemExit(0)
    main()
