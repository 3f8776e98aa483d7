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
