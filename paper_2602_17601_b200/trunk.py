"""Chain plant of the closed-loop tracking configuration (BASELINE cfg2), on
the device.

Mirror of the reference plant (``trunk.py:23-187``): ``ChainConfig`` keeps the
reference's fields, defaults and validation; ``DevicePlant.step`` advances a
device-resident state by one controller period with the sm_100a kernel
``gm_trunk_step`` (semi-implicit Euler substeps, fp64, the reference's term
order), so a closed loop never round-trips the state through the host.  The
plant is the environment of the hot path, not part of it; it
exists here for the device-resident closed loop of SURVEY.md 8(f), rank 1.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from . import device as _dev
from ._runtime import addr
from .graph import SystemState, chain_topology


@dataclass
class ChainConfig:
    """Plant parameters (``trunk.py:23-113``)."""

    node_count: int = 4
    node_mass: float = 0.08
    coupling_stiffness: float = 300.0
    coupling_damping: float = 2.0
    bend_stiffness: float = 25.0
    rest_length: float = 0.15
    gravity: tuple = (0.0, 0.0, -9.81)
    tendon_directions: np.ndarray | None = None
    tendon_nodes: tuple | None = None
    u_max: float = 8.0
    dt_sim: float = 1e-3
    dt: float = 0.01

    def __post_init__(self):
        if self.node_count < 2:
            raise ValueError("need at least a base and one moving node")
        if self.node_mass <= 0 or self.coupling_stiffness <= 0:
            raise ValueError("mass and coupling stiffness must be positive")
        if self.coupling_damping < 0 or self.bend_stiffness < 0:
            raise ValueError("damping and bend stiffness must be nonnegative")
        if self.dt_sim <= 0 or self.dt <= 0:
            raise ValueError("time steps must be positive")
        ratio = self.dt / self.dt_sim
        if abs(ratio - round(ratio)) > 1e-9:
            raise ValueError("dt_sim must divide dt")
        if self.tendon_directions is None:  # three antagonistic pairs, 60 degrees apart
            angles = np.deg2rad([0, 60, 120, 180, 240, 300])
            self.tendon_directions = np.stack([np.cos(angles), np.sin(angles), np.zeros(6)], axis=1)
        else:
            self.tendon_directions = np.asarray(self.tendon_directions, dtype=float)
        if self.tendon_nodes is None:
            moving = tuple(range(1, self.node_count))
            self.tendon_nodes = tuple(moving for _ in range(self.n_u))
        if len(self.tendon_nodes) != self.n_u:
            raise ValueError("one attachment set per tendon required")
        for nodes in self.tendon_nodes:
            for i in nodes:
                if not 1 <= i < self.node_count:
                    raise ValueError("tendons attach to moving nodes only")
        self.gravity = tuple(float(v) for v in self.gravity)

    @property
    def n_u(self) -> int:
        return self.tendon_directions.shape[0]

    @property
    def substeps(self) -> int:
        return int(round(self.dt / self.dt_sim))

    def rest_positions(self) -> np.ndarray:
        out = np.zeros((self.node_count, 3))
        out[:, 2] = -self.rest_length * np.arange(self.node_count)
        return out

    def rest_state(self) -> SystemState:
        arr = np.zeros((self.node_count, 6))
        arr[:, :3] = self.rest_positions()
        return SystemState(arr)

    def tendon_force_map(self) -> np.ndarray:
        """(M, 3, n_u) tensions -> per-node forces (``trunk.py:96-104``)."""
        out = np.zeros((self.node_count, 3, self.n_u))
        for t, nodes in enumerate(self.tendon_nodes):
            w = 1.0 / len(nodes)
            for i in nodes:
                out[i, :, t] = w * self.tendon_directions[t]
        return out

    def to_dict(self) -> dict:
        d = asdict(self)
        d["tendon_directions"] = self.tendon_directions.tolist()
        d["tendon_nodes"] = [list(n) for n in self.tendon_nodes]
        return d


class DevicePlant:
    """``step_state_array`` (``trunk.py:148-160``) on the device for one or a
    batch of plants: states (M, 6) or (B, M, 6) fp64 device tensors."""

    def __init__(self, cfg: ChainConfig, topo=None, device=None):
        self.cfg = cfg
        self.topo = topo if topo is not None else chain_topology(cfg.node_count)
        self.eng = eng = _dev.engine(self.topo, None, device)
        f64 = np.float64
        self.rest = eng.h2d(cfg.rest_positions(), f64)
        self.fmap = eng.h2d(cfg.tendon_force_map(), f64)
        self.gravity = np.ascontiguousarray(cfg.gravity, dtype=f64)  # host array (ABI)
        self.bad = eng.zeros((1,), np.int32)

    def step(self, X, U, clip_inputs: bool = True, out=None):
        """One controller period; returns the new state tensor (``out`` if given)."""
        torch, eng, cfg = self.eng.torch, self.eng, self.cfg
        X = X if hasattr(X, "data_ptr") and not isinstance(X, np.ndarray) else \
            torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).to(eng.device)
        U = U if hasattr(U, "data_ptr") and not isinstance(U, np.ndarray) else \
            torch.from_numpy(np.ascontiguousarray(np.asarray(U, dtype=np.float64))).to(eng.device)
        X = X.contiguous()
        U = U.contiguous()
        B = 1 if X.dim() == 2 else int(X.shape[0])
        if out is None:
            out = torch.empty_like(X)
        eng.ctx.call("gm_trunk_step", B, cfg.node_count, cfg.n_u, cfg.substeps, float(cfg.dt_sim),
                     float(cfg.node_mass), float(cfg.coupling_stiffness), float(cfg.coupling_damping),
                     float(cfg.bend_stiffness), float(cfg.rest_length), addr(self.gravity),
                     addr(self.rest), addr(self.fmap), float(cfg.u_max), 1 if clip_inputs else 0,
                     addr(X), addr(U), addr(out), addr(self.bad), eng.stream_ptr())
        return out

    def check_finite(self):
        """Raise like the reference (``trunk.py:158-159``) if any step blew up."""
        if int(self.bad.item()):
            self.bad.zero_()
            raise FloatingPointError("simulation blew up: non-finite state")

    def settle(self, seconds: float = 3.0, u=None):
        """``settle`` (``trunk.py:181-187``): constant input from rest."""
        cfg = self.cfg
        u = np.zeros(cfg.n_u) if u is None else np.asarray(u, dtype=float)
        x = self.eng.h2d(cfg.rest_state().array, np.float64)
        ud = self.eng.h2d(u, np.float64)
        for _ in range(int(round(seconds / cfg.dt))):
            x = self.step(x, ud)
        self.check_finite()
        return x
