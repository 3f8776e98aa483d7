"""Engine / plan lifecycle on the GPU: captured step graphs stay correct when
the model is edited or replaced, plans die with their spec, BatchedMpc honours
the per-instance previous input in the fallback (advisor findings, round 1).
"""

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _steps(pkg, model, topo, spec, x, cfg, n=3):
    st = pkg.mpc_init(x, cfg, 6)
    out = None
    for _ in range(n):  # eager run, capture, graph replay
        out = pkg.mpc_step(model, topo, spec, x, st, cfg)
    return out


def _oracle_u(model, topo, spec, x0, N):
    from oracle import ref_port as O

    return O.mpc_step(model, topo, spec, x0, np.tile(x0, (N + 1, 1, 1)), np.zeros((N, 6)), N)


def test_model_edit_after_capture_is_honoured():
    """In-place weight edits (same dims) are copied into the buffers the
    captured graph reads; a model with other layer dims on the same topology
    re-allocates the buffers, bumps the model generation and drops the
    captured graphs (device.Engine.bind_model)."""
    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import device, workloads
    from paper_2602_17601_b200._runtime import lib
    from paper_2602_17601_b200.mpc import get_plan

    N = 8
    topo, model, states, inputs, spec = workloads.scaling_problem(30, N, 0.01, 4)
    spec.freeze()
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(states[0])
    u, st = _steps(pkg, model, topo, spec, x, cfg)
    eng = device.engine(topo, model)
    plan = get_plan(eng, spec, N, 6, 6, cfg, True)
    assert plan.graph is not None  # the whole step is a captured graph now
    gen0 = lib().gm_model_generation(eng.ctx.handle)

    # 1. in-place edit, same dims: same generation, graph kept, new weights used
    rng = np.random.default_rng(1)
    for W in model.phi.weights + model.psi.weights:
        W[...] *= 1.0 + 0.3 * rng.standard_normal(W.shape)
    u1, st1 = _steps(pkg, model, topo, spec, x, cfg, n=1)
    assert lib().gm_model_generation(eng.ctx.handle) == gen0
    assert get_plan(eng, spec, N, 6, 6, cfg, True) is plan
    ref = _oracle_u(model, topo, spec, states[0], N)
    assert st1.last_status.value == ref["status"]
    assert np.max(np.abs(u1.u - ref["u_applied"])) <= TOL * max(1.0, np.max(np.abs(ref["u_applied"])))
    assert np.max(np.abs(u1.u - u.u)) > 1e-6  # the edit changed the answer

    # 2. a model with other hidden widths on the same topology
    m2 = pkg.init_model(3, 6, 0.01, np.random.default_rng(9), n_m=16, psi_hidden=(24, 24),
                        phi_hidden=(48, 40), out_scale=0.05)
    u2, st2 = _steps(pkg, m2, topo, spec, x, cfg)
    assert lib().gm_model_generation(eng.ctx.handle) > gen0
    ref2 = _oracle_u(m2, topo, spec, states[0], N)
    assert st2.last_status.value == ref2["status"]
    assert np.max(np.abs(u2.u - ref2["u_applied"])) <= TOL * max(1.0, np.max(np.abs(ref2["u_applied"])))

    # 3. and back (dims change again): correct again
    u3, _ = _steps(pkg, model, topo, spec, x, cfg)
    assert np.max(np.abs(u3.u - ref["u_applied"])) <= TOL * max(1.0, np.max(np.abs(ref["u_applied"])))


def test_plans_die_with_their_spec():
    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import device, workloads

    N = 6
    topo, model, states, inputs, spec0 = workloads.scaling_problem(12, N, 0.01, 5)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x = pkg.SystemState(states[0])
    eng = device.engine(topo, model)

    def n_plans():
        return sum(1 for k in eng.cache if isinstance(k, tuple) and k and k[0] == "plan")

    base = n_plans()
    for _ in range(5):  # a fresh frozen spec per call (a loop that re-freezes)
        spec = pkg.OcpSpec(topo, N, spec0.q.copy(), spec0.x_ref.copy(), spec0.r.copy(),
                           spec0.u_ref.copy(), spec0.input_constraints,
                           list(spec0.state_constraints)).freeze()
        _steps(pkg, model, topo, spec, x, cfg, n=2)
        del spec
        gc.collect()
    assert n_plans() <= base + 1


def test_batched_fallback_holds_previous_input():
    """BatchedMpc with the hold-previous-input policy applies each instance's
    own last input when its QP fails, zeros when none is given (mpc.py:163-170)."""
    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200.batch import BatchedMpc
    from paper_2602_17601_b200.condensing import OcpSpec, StateConstraint
    from paper_2602_17601_b200.errors import ConfigurationError
    from tests.golden_io import mpc_branch_cases

    bc = mpc_branch_cases()
    N, M, B = bc.spec.horizon, bc.topo.node_count, 3
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    bm = BatchedMpc(bc.model, bc.topo, bc.bad, cfg, B)
    x0 = np.stack([bc.x_seq[0]] * B)
    ls = np.repeat(x0[:, None], N + 1, axis=1)
    li = np.zeros((B, N, 6))
    xr = np.repeat(x0[:, :, None], N + 1, axis=2)
    prev = np.arange(B * 6, dtype=float).reshape(B, 6) * 0.1
    res = bm.step(x0, ls, li, xr, last_applied=prev)
    assert all(s.value == "primal_infeasible" for s in res.status)
    assert np.array_equal(res.u_applied, prev)
    res = bm.step(x0, ls, li, xr)
    assert np.array_equal(res.u_applied, np.zeros((B, 6)))
    with pytest.raises(ConfigurationError):
        BatchedMpc(bc.model, bc.topo, bc.spec, pkg.MpcConfig(horizon=N, dt=0.01, sqp_iterations=2), B)
