"""GPU tests of the device-resident closed loop (BASELINE cfg2): the chain
plant kernel and the controller + plant loop against golden vectors made by
the reference's own trunk plant, tracking provider and run_closed_loop
(oracle/make_golden.py cfg2)."""

import numpy as np
import pytest

from oracle import ref_port as O
from tests.golden_io import load, model_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load("cfg2_closed_loop")


def test_device_plant_matches_reference(g):
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

    M = g["x0"].shape[0]
    plant = DevicePlant(ChainConfig(node_count=M))
    out = plant.step(g["plant_in"], g["plant_u"]).cpu().numpy()
    assert np.max(np.abs(out - g["plant_out"])) <= 1e-12


def test_device_plant_batched_matches_oracle(g):
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

    M = 37
    cfg = ChainConfig(node_count=M)
    plant = DevicePlant(cfg)
    P = O.trunk_params(M)
    rng = np.random.default_rng(1)
    X = np.stack([cfg.rest_state().array + 0.02 * rng.standard_normal((M, 6)) for _ in range(3)])
    U = rng.uniform(-1.0, 9.0, (3, 6))
    out = plant.step(X, U).cpu().numpy()
    for b in range(3):
        ref = O.trunk_step(P, X[b], U[b])
        assert np.max(np.abs(out[b] - ref)) <= 1e-12


def test_device_plant_settle_matches_oracle():
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

    cfg = ChainConfig(node_count=12)
    x = DevicePlant(cfg).settle(0.2).cpu().numpy()
    P = O.trunk_params(12)
    ref = cfg.rest_state().array
    for _ in range(20):
        ref = O.trunk_step(P, ref, np.zeros(6))
    assert np.max(np.abs(x - ref)) <= 1e-11


def test_device_closed_loop_matches_reference(g):
    """Controller and plant alternate on the device; inputs, statuses and the
    plant trajectory follow the reference's closed loop."""
    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200.graph import chain_topology
    from paper_2602_17601_b200.tracking import (TrackingWeights, circle_reference,
                                                 run_closed_loop_device, tracking_spec_provider)
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

    M = g["x0"].shape[0]
    topo = chain_topology(M)
    model = model_from(g, "m_")
    plant = DevicePlant(ChainConfig(node_count=M), topo)
    cfg = pkg.MpcConfig(horizon=10, dt=0.01)
    prov = tracking_spec_provider(topo, cfg, pkg.SystemState(g["x0"]),
                                  circle_reference(0.04, 8.0, g["center"]), TrackingWeights(), 6, 8.0)
    log = run_closed_loop_device(plant, model, topo, prov, g["x0"], 6, cfg)
    assert [s.value for s in log.statuses] == [str(s) for s in g["statuses"]]
    assert np.max(np.abs(log.iterations - g["iterations"])) <= 1
    assert np.max(np.abs(log.inputs - g["inputs"])) <= 1e-4 * 8.0
    assert np.max(np.abs(log.states - g["states"])) <= 1e-6
