"""Closed-loop reference tracking on the device (BASELINE cfg2).

Mirrors the reference's tracking stack -- ``circle_reference``
(``references.py:12-30``), ``TrackingWeights`` and ``tracking_spec_provider``
(``experiments.py:90-139``), ``run_closed_loop`` / ``run_tracking``
(``mpc.py:224-264``, ``experiments.py:347-379``) -- with the controller step
(``mpc_step``) and the chain plant (``trunk.DevicePlant``) both on the GPU: the
state stays in HBM between steps, and per step only the moving part of the
OCP (the reference trajectory x_ref, 8 KB per node block row) is uploaded.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .condensing import OcpSpec, stage_input_box
from .graph import SystemState
from .mpc import ClosedLoopLog, MpcConfig, mpc_init, mpc_step
from .trunk import ChainConfig, DevicePlant


def circle_reference(radius: float, period: float, center):
    """x-y circle from angle 0 with tangential speed 2 pi r / period
    (``references.py:12-30``): t -> (positions, velocities)."""
    center = np.asarray(center, dtype=float)
    omega = 2.0 * np.pi / period

    def ref(t):
        t = np.asarray(t, dtype=float)
        ang = omega * t
        pos = np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros_like(ang)], axis=-1) + center
        vel = np.stack([-radius * omega * np.sin(ang), radius * omega * np.cos(ang), np.zeros_like(ang)],
                       axis=-1)
        return pos, vel

    return ref


@dataclass
class TrackingWeights:
    """``experiments.py:90-104``."""

    q_pos: tuple = (500.0, 500.0, 100.0)
    q_vel: tuple = (0.5, 0.5, 0.5)
    r_diag: float = 2e-4
    rest_q_pos: float = 0.0

    def node_block(self, on_target: bool) -> np.ndarray:
        q = np.zeros(6)
        if on_target:
            q[:3] = self.q_pos
            q[3:] = self.q_vel
        else:
            q[:3] = self.rest_q_pos
        return np.diag(q)


class _StaticToken:
    """Identity of the part of a tracking OCP that does not change between
    steps (costs, u_ref, input box); ``device_spec`` caches its upload under it
    and refreshes only x_ref."""


def tracking_spec_provider(topo, cfg: MpcConfig, rest_state: SystemState, ee_reference,
                           weights: TrackingWeights, n_u: int, u_max: float, target_node: int | None = None):
    """``experiments.py:107-139``: the target node follows the curve, the others
    see their rest pose.  Every spec shares the same (frozen) cost arrays and
    carries the provider's static token."""
    M = topo.node_count
    N = cfg.horizon
    target = M - 1 if target_node is None else target_node
    q = np.zeros((M, N + 1, 6, 6))
    for i in range(M):
        q[i, :] = weights.node_block(i == target)
    r = np.tile(np.eye(n_u) * weights.r_diag, (N, 1, 1))
    u_ref = np.zeros((N, n_u))
    box = stage_input_box(n_u, 0.0, u_max)
    input_cons = [box] * N
    rest_arr = np.asarray(rest_state.array, dtype=float)
    x_base = np.tile(rest_arr[:, None, :], (1, N + 1, 1))
    stage_offsets = np.arange(N + 1) * cfg.dt
    for a in (q, r, u_ref):
        a.flags.writeable = False
    token = _StaticToken()

    def provider(t: int, _mpc_state) -> OcpSpec:
        x_ref = x_base.copy()
        pos, vel = ee_reference(t * cfg.dt + stage_offsets)
        x_ref[target, :, :3] = pos
        x_ref[target, :, 3:] = vel
        spec = OcpSpec(topo, N, q, x_ref, r, u_ref, input_cons, [])
        object.__setattr__(spec, "_static_token", token)
        return spec

    return provider


class _DeviceState:
    """A measured state that already lives on the device ((M, nx) tensor)."""

    def __init__(self, t):
        self.array = t


def run_closed_loop_device(plant: DevicePlant, model, topo, spec_provider, x0, n_steps: int,
                           cfg: MpcConfig) -> ClosedLoopLog:
    """``run_closed_loop`` (``mpc.py:224-264``) with a device plant: controller
    and plant alternate on the GPU, the state never leaves HBM; states are
    copied to the host once, after the loop."""
    torch = plant.eng.torch
    x = x0 if hasattr(x0, "data_ptr") else plant.eng.h2d(np.asarray(
        x0.array if hasattr(x0, "array") else x0, dtype=float), np.float64)
    n_u = spec_provider(0, None).n_u if callable(spec_provider) else spec_provider.n_u
    state = mpc_init(SystemState(x.cpu().numpy()), cfg, n_u)
    traj = [x]
    us, statuses, iters, timings, xrefs = [], [], [], [], []
    for t in range(n_steps):
        spec = spec_provider(t, state) if callable(spec_provider) else spec_provider
        u, state = mpc_step(model, topo, spec, _DeviceState(x), state, cfg)
        u_dev = state.device_value("last_applied")
        if u_dev is None or isinstance(u_dev, np.ndarray):
            u_dev = plant.eng.h2d(u.u, np.float64)
        x = plant.step(x, u_dev)
        traj.append(x)
        us.append(u.u)
        statuses.append(state.last_status)
        iters.append(state.last_iterations)
        tm = state.last_timing
        timings.append((tm.linearize_ms, tm.condense_ms, tm.solve_ms, tm.total_ms))
        xrefs.append(spec.x_ref[:, 0, :3])
    plant.check_finite()
    states = torch.stack(traj).cpu().numpy()
    n_p = states.shape[-1] // 2
    errs = np.linalg.norm(states[:-1, :, :n_p] - np.stack(xrefs), axis=-1) if n_steps else \
        np.zeros((0, states.shape[1]))
    return ClosedLoopLog(states, np.asarray(us).reshape(n_steps, n_u), statuses,
                         np.asarray(iters, dtype=int), np.asarray(timings).reshape(n_steps, 4), errs, cfg.dt)


def run_tracking_device(plant_cfg: ChainConfig, model, mpc_cfg: MpcConfig, ee_reference, n_steps: int,
                        weights: TrackingWeights | None = None, settle_s: float = 3.0):
    """``run_tracking`` (``experiments.py:347-379``) on the device; returns
    (log, wall seconds of the closed loop)."""
    from .graph import chain_topology

    topo = chain_topology(plant_cfg.node_count)
    plant = DevicePlant(plant_cfg, topo)
    weights = weights or TrackingWeights()
    x0 = plant.settle(settle_s)
    rest = SystemState(x0.cpu().numpy())
    provider = tracking_spec_provider(topo, mpc_cfg, rest, ee_reference, weights, plant_cfg.n_u,
                                      plant_cfg.u_max)
    t0 = time.perf_counter()
    log = run_closed_loop_device(plant, model, topo, provider, x0, n_steps, mpc_cfg)
    return log, time.perf_counter() - t0


@dataclass
class ObstacleScenario:
    """A sphere approaching a target point along a line, holding, then
    retreating (``experiments.py:142-183``)."""

    target_point: np.ndarray
    approach_from: np.ndarray
    radius: float = 0.05
    margin: float = 0.01
    start_distance: float = 0.5
    approach_time: float = 4.0
    hold_time: float = 3.0
    retreat_time: float = 4.0
    start_delay: float = 1.0
    constrained_nodes: tuple = ()
    activation_factor: float = 2.5
    rho1: float = 1e3
    rho2: float = 1e4

    def center(self, t):
        """Sphere centre at time(s) t (``experiments.py:162-179``)."""
        t = np.asarray(t, dtype=float)
        d0 = self.start_distance
        t1 = self.start_delay
        t2 = t1 + self.approach_time
        t3 = t2 + self.hold_time
        t4 = t3 + self.retreat_time
        dist = np.where(t < t1, d0,
                        np.where(t < t2, d0 * (t2 - t) / self.approach_time,
                                 np.where(t < t3, 0.0, np.where(t < t4, d0 * (t - t3) / self.retreat_time, d0))))
        return np.asarray(self.target_point, dtype=float) + dist[..., None] * np.asarray(self.approach_from,
                                                                                      dtype=float)

    @property
    def total_time(self) -> float:
        return self.start_delay + self.approach_time + self.hold_time + self.retreat_time


def obstacle_spec_provider(topo, cfg: MpcConfig, rest_state: SystemState, scenario: ObstacleScenario,
                           weights: TrackingWeights, n_u: int, u_max: float):
    """Rest-pose regulation plus time-varying avoidance half-spaces
    (``experiments.py:186-238``): per constrained node and stage k = 1..N, a
    soft row -n^T p <= -(r + margin) - n^T c_k when the predicted position is
    within activation range of the sphere, n the unit vector from the centre
    to the prediction.  The predictions are the controller's own shifted plan
    (``MpcState.lin_states``); only the constrained nodes' positions are read
    back from the device.""" 
    from .condensing import StateConstraint

    M = topo.node_count
    N = cfg.horizon
    q = np.zeros((M, N + 1, 6, 6))
    diag = np.zeros(6)
    diag[:3] = weights.q_pos
    diag[3:] = weights.q_vel
    q[:, :] = np.diag(diag)
    r = np.tile(np.eye(n_u) * weights.r_diag, (N, 1, 1))
    u_ref = np.zeros((N, n_u))
    input_cons = [stage_input_box(n_u, 0.0, u_max)] * N
    rest_arr = np.asarray(rest_state.array, dtype=float)
    x_ref = np.tile(rest_arr[:, None, :], (1, N + 1, 1))
    for a in (q, r, u_ref, x_ref):
        a.flags.writeable = False
    r_active = scenario.activation_factor * (scenario.radius + scenario.margin)
    r_con = scenario.radius + scenario.margin
    stage_offsets = np.arange(N + 1) * cfg.dt
    nodes = tuple(int(i) for i in scenario.constrained_nodes)

    def predicted(mpc_state):
        """(N+1 or 1, len(nodes), 3) predicted positions of the constrained nodes."""
        if mpc_state is None:
            return rest_arr[None, nodes, :3]
        ls = mpc_state.lin_states
        if hasattr(ls, "data_ptr") and not isinstance(ls, np.ndarray):
            return ls[:, list(nodes), :3].cpu().numpy()
        ls = np.asarray(ls, dtype=float)
        return ls[:, nodes, :3] if ls.ndim == 3 else ls[None, nodes, :3]

    def provider(t: int, mpc_state) -> OcpSpec:
        pred = predicted(mpc_state)
        centers = scenario.center(t * cfg.dt + stage_offsets)  # (N+1, 3)
        cons = []
        for k in range(1, N + 1):
            for a, node in enumerate(nodes):
                p_hat = pred[min(k, len(pred) - 1), a]
                rel = p_hat - centers[k]
                dist = float(np.linalg.norm(rel))
                if dist > r_active:
                    continue
                n_hat = rel / max(dist, 1e-9)
                row = np.zeros((1, 6))
                row[0, :3] = -n_hat
                bound = np.array([-r_con - float(n_hat @ centers[k])])
                cons.append(StateConstraint(node, k, row, bound, soft=True, rho1=scenario.rho1,
                                            rho2=scenario.rho2))
        # the constraint rows change every step: no static token (device_spec
        # rebuilds the device copy), unlike the tracking provider
        return OcpSpec(topo, N, q, x_ref, r, u_ref, input_cons, cons)

    return provider
