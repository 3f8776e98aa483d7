"""The drop-in boundary against the REAL reference: the unmodified reference
``gnnmpc.mpc.mpc_step`` (installed in ``baseline/_ref`` by
``pip install --no-index --target baseline/_ref``), once on its own CPU
stages and once with its stage globals rebound to the B200 path
(``paper_2602_17601_b200.integrate.install``).  The
reference's own control logic -- SQP loop, damping, fallback, input filter,
shift -- runs in both; only the stages differ.  Also the reference's
``Linearizer`` plug-in point (``mpc.py:23``, ``:82-87``) with the GPU
linearisation as the callable.

Skipped when ``baseline/_ref`` is absent (it is git-ignored; it travels to the
GPU box with the working tree).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
TOL = 1e-4


@pytest.fixture(scope="module")
def ref():
    if not (REF / "gnnmpc" / "mpc.py").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    try:
        import gnnmpc.condensing as rc
        import gnnmpc.experiments as rex
        import gnnmpc.graph as rgr
        import gnnmpc.mpc as rm
        import gnnmpc.qpsolver as rq
    finally:
        sys.path.remove(str(REF))
    assert Path(rm.__file__).resolve().is_relative_to(REF.resolve())
    return dict(rc=rc, rex=rex, rgr=rgr, rm=rm, rq=rq)


def _seq(rm, rgr, model, topo, specs, xs, cfg):
    st = rm.mpc_init(rgr.SystemState(xs[0]), cfg, 6)
    out = []
    for spec, x in zip(specs, xs):
        u, st = rm.mpc_step(model, topo, spec, rgr.SystemState(x), st, cfg)
        out.append((np.array(u.u), st))
    return out


def _compare(a, b, info):
    for t, ((ua, sa), (ub, sb)) in enumerate(zip(a, b)):
        i = (info, t)
        assert sa.last_status == sb.last_status, i
        assert abs(sa.last_iterations - sb.last_iterations) <= 2, i
        scale = max(1.0, float(np.max(np.abs(ub))))
        assert float(np.max(np.abs(ua - ub))) / scale <= TOL, i
        xs = max(1.0, float(np.max(np.abs(sb.lin_states))))
        assert float(np.max(np.abs(np.asarray(sa.lin_states) - sb.lin_states))) / xs <= TOL, i
        assert float(np.max(np.abs(np.asarray(sa.lin_inputs) - sb.lin_inputs))) / scale <= TOL, i


@pytest.mark.parametrize("variant", ["rti", "sqp2damp", "filter", "fallback"])
def test_unmodified_reference_mpc_step_on_b200_stages(ref, variant):
    from paper_2602_17601_b200 import integrate

    rc, rex, rgr, rm = ref["rc"], ref["rex"], ref["rgr"], ref["rm"]
    N = 10
    topo, model, states, inputs, spec = rex._scaling_problem(40, N, 0.01, 0)
    rng = np.random.default_rng(3)
    xs = [states[0] + 0.002 * rng.standard_normal(states[0].shape) for _ in range(3)]
    specs = [spec] * 3
    kw = {}
    if variant == "sqp2damp":
        kw = dict(sqp_iterations=2, sqp_damping=0.5)
    elif variant == "filter":
        kw = dict(input_filter_tau=0.05)
    elif variant == "fallback":
        rows = np.zeros((2, 6))
        rows[0, 2], rows[1, 2] = 1.0, -1.0
        bad = rc.OcpSpec(topo, N, spec.q, spec.x_ref, spec.r, spec.u_ref, spec.input_constraints,
                         list(spec.state_constraints)
                         + [rc.StateConstraint(0, 1, rows, np.array([-100.0, -100.0]))])
        specs = [spec, bad, spec]
    cfg = rm.MpcConfig(horizon=N, dt=0.01, **kw)
    cpu = _seq(rm, rgr, model, topo, specs, xs, cfg)
    saved = integrate.install(rm)
    try:
        assert rm.condense_gammas is not saved["condense_gammas"]
        gpu = _seq(rm, rgr, model, topo, specs, xs, cfg)
    finally:
        integrate.uninstall(rm, saved)
    assert rm.solve_qp is saved["solve_qp"]
    if variant == "fallback":
        assert gpu[1][1].last_status.value == "primal_infeasible"
    _compare(gpu, cpu, variant)


def test_reference_linearizer_plugin_point(ref):
    """Stage 1 only: the GPU linearisation as the reference's Linearizer
    callable; the reference's own CPU stages 2-4 consume its blocks."""
    import paper_2602_17601_b200 as pkg

    rex, rgr, rm = ref["rex"], ref["rgr"], ref["rm"]
    N = 10
    topo, model, states, inputs, spec = rex._scaling_problem(40, N, 0.01, 1)
    cfg = rm.MpcConfig(horizon=N, dt=0.01)
    xs = [states[0]] * 2
    cpu = _seq(rm, rgr, model, topo, [spec] * 2, xs, cfg)

    def lin(s, u):
        d = pkg.linearize_trajectory(model, topo, s, u)
        return rm.LinearizedDynamics(topo, d.horizon, np.array(d.a_self), np.array(d.a_nbr),
                                     np.array(d.b), np.array(d.c))

    gpu = _seq(rm, rgr, lin, topo, [spec] * 2, xs, cfg)
    _compare(gpu, cpu, "plugin")
