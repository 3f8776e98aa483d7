"""Obstacle-avoidance OCP provider: per-step soft
half-spaces built from the controller's own predicted positions
(experiments.py:142-238), pinned to the reference's output
(tests/golden/obstacle_provider.npz, made by oracle/make_golden.py obstacle),
and -- on the GPU -- a few receding-horizon steps through mpc_step against the
CPU oracle with the moving constraint rows."""

from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "obstacle_provider.npz"
M, N = 12, 10


class _State:
    def __init__(self, ls):
        self.lin_states = ls


def _provider(d):
    from paper_2602_17601_b200.graph import SystemState, chain_topology
    from paper_2602_17601_b200.mpc import MpcConfig
    from paper_2602_17601_b200.tracking import ObstacleScenario, TrackingWeights, obstacle_spec_provider
    from paper_2602_17601_b200.trunk import ChainConfig

    x0 = d["x0"]
    mid = 0.5 * (x0[-1, :3] + x0[-2, :3])
    scen = ObstacleScenario(target_point=mid + np.array([0.05, 0.0, 0.0]), approach_from=np.array([1.0, 0.0, 0.0]),
                            constrained_nodes=(M - 1, M - 2, 5), start_distance=0.3, approach_time=2.0,
                            hold_time=1.0, retreat_time=2.0, start_delay=0.2)
    pc = ChainConfig(node_count=M)
    topo = chain_topology(M)
    cfg = MpcConfig(horizon=N, dt=0.01)
    prov = obstacle_spec_provider(topo, cfg, SystemState(x0), scen, TrackingWeights(), pc.n_u, pc.u_max)
    return topo, cfg, scen, prov, pc


def test_obstacle_provider_matches_reference():
    d = np.load(GOLD)
    topo, cfg, scen, prov, pc = _provider(d)
    assert np.allclose(scen.center(np.arange(0, 6.0, 0.01)), d["centers"], rtol=0, atol=1e-15)
    for key in d["cases"]:
        t, with_state = (int(v) for v in str(key).split("_"))
        st = _State(d[f"pred_{t}"]) if with_state else None
        spec = prov(t, st)
        cons = spec.state_constraints
        assert np.array_equal(np.array([c.node for c in cons], dtype=np.int64), d[f"nodes_{key}"]), key
        assert np.array_equal(np.array([c.stage for c in cons], dtype=np.int64), d[f"stages_{key}"]), key
        if cons:
            assert np.allclose(np.array([c.c for c in cons]).reshape(-1, 6), d[f"rows_{key}"], rtol=0, atol=1e-14)
            assert np.allclose(np.array([c.d for c in cons]).reshape(-1), d[f"bounds_{key}"], rtol=0, atol=1e-14)
            assert all(c.soft for c in cons)
            assert np.array_equal(np.array([[c.rho1, c.rho2] for c in cons]), d[f"rho_{key}"])
        for name in ("q", "x_ref", "r", "u_ref"):
            assert np.array_equal(getattr(spec, name), d[name]), name


@pytest.mark.gpu
def test_obstacle_receding_horizon_matches_oracle():
    """Five mpc_step calls inside the obstacle's hold window (t = 230..234),
    constraint rows rebuilt from the GPU plan each step, against the oracle
    fed the same specs; also checks that specs rebuilt every step reuse one
    step plan per row layout (no per-step device allocations)."""
    import paper_2602_17601_b200 as pkg
    from oracle import ref_port as O
    from paper_2602_17601_b200 import device
    from paper_2602_17601_b200.gnn import init_model

    d = np.load(GOLD)
    topo, cfg, scen, prov, pc = _provider(d)
    model = init_model(3, 6, 0.01, np.random.default_rng(3), n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64),
                       out_scale=0.05)
    x = pkg.SystemState(d["x0"])
    st = pkg.mpc_init(x, cfg, pc.n_u)
    ref_ls = np.repeat(d["x0"][None], N + 1, axis=0)
    ref_li = np.zeros((N, pc.n_u))
    eng = device.engine(topo, model)
    plans0 = None
    for step, t in enumerate(range(230, 235)):
        spec = prov(t, st)
        ref_spec = spec
        u, st = pkg.mpc_step(model, topo, spec, x, st, cfg)
        ref = O.mpc_step(model, topo, ref_spec, d["x0"], ref_ls, ref_li, N)
        assert st.last_status.value == ref["status"], (t, st.last_status, ref["status"])
        scale = max(1.0, float(np.max(np.abs(ref["u_applied"]))))
        assert float(np.max(np.abs(u.u - ref["u_applied"]))) / scale <= 1e-4, t
        ref_ls, ref_li = ref["lin_states"], ref["lin_inputs"]
        n_plans = sum(1 for k in eng.cache if isinstance(k, tuple) and k[:1] == ("plan",))
        if plans0 is None:
            plans0 = n_plans
        assert n_plans <= plans0 + 3  # one plan per distinct row layout, not per step
