"""GNN dynamics model and its linearisation -- reference-compatible API.

Mirrors ``gnnmpc/gnn.py``: ``Normalization`` / ``GnnModel`` / ``init_model``
(``:26-104``), ``step_array`` / ``gnn_step`` / ``rollout`` (``:153-182``),
``LinearizedDynamics`` (``:185-234``), ``linearize_stage`` /
``linearize_trajectory`` (``:301-321``) and the JSON model format
(``:324-378``).  The compute runs in the fused sm_100a kernel K-LIN
(``csrc/k_linearize.cu``) through the C ABI; results come back as a
``LinearizedDynamics`` whose blocks live on the GPU (fp32) and are
materialised to NumPy fp64 only when a caller reads them.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from . import device as _dev
from .graph import GraphTopology, InputVector, SystemState, Trajectory
from .mlp import MlpParams, mlp_init


@dataclass
class Normalization:
    state_mean: np.ndarray
    state_scale: np.ndarray
    input_mean: np.ndarray
    input_scale: np.ndarray

    def __post_init__(self):
        for name in ("state_mean", "state_scale", "input_mean", "input_scale"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=float))
        if np.any(self.state_scale <= 0) or np.any(self.input_scale <= 0):
            raise ValueError("normalization scales must be positive")

    @classmethod
    def identity(cls, n_state: int, n_u: int) -> "Normalization":
        return cls(np.zeros(n_state), np.ones(n_state), np.zeros(n_u), np.ones(n_u))


@dataclass
class GnnModel:
    """Edge MLP psi, node MLP phi, sampling period (validation ``gnn.py:56-71``)."""

    psi: MlpParams
    phi: MlpParams
    dt: float
    n_p: int
    n_u: int
    n_m: int
    normalization: Normalization

    def __post_init__(self):
        nx = 2 * self.n_p
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.psi.in_dim != nx:
            raise ValueError(f"psi input dim {self.psi.in_dim} != node state dim {nx}")
        if self.psi.out_dim != self.n_m:
            raise ValueError("psi output dim != n_m")
        if self.phi.in_dim != nx + self.n_m + self.n_u:
            raise ValueError("phi input dim != n_state + n_m + n_u")
        if self.phi.out_dim != self.n_p:
            raise ValueError("phi output dim != n_p")
        if self.normalization.state_mean.shape != (nx,):
            raise ValueError("normalization state stats must have node-state length")
        if self.normalization.input_mean.shape != (self.n_u,):
            raise ValueError("normalization input stats must have input length")

    @property
    def n_state(self) -> int:
        return 2 * self.n_p

    def freeze(self) -> "GnnModel":
        """Make the parameters immutable (arrays read-only, layer lists
        tuples).  A frozen model is re-checked by identity instead of by a
        byte fingerprint of its ~8 k parameters on every ``mpc_step`` (the
        reference reads the arrays on every call; an unfrozen model keeps
        that semantics, in-place edits included)."""
        for mlp in (self.psi, self.phi):
            for a in list(mlp.weights) + list(mlp.biases):
                a.flags.writeable = False
            mlp.weights = tuple(mlp.weights)
            mlp.biases = tuple(mlp.biases)
        nrm = self.normalization
        for a in (nrm.state_mean, nrm.state_scale, nrm.input_mean, nrm.input_scale):
            a.flags.writeable = False
        object.__setattr__(self, "_frozen", (id(self.psi), id(self.phi), id(nrm), self.dt))
        return self

    def copy(self) -> "GnnModel":
        nrm = self.normalization
        return GnnModel(self.psi.copy(), self.phi.copy(), self.dt, self.n_p, self.n_u, self.n_m,
                        Normalization(nrm.state_mean.copy(), nrm.state_scale.copy(),
                                      nrm.input_mean.copy(), nrm.input_scale.copy()))


def init_model(n_p: int, n_u: int, dt: float, rng: np.random.Generator, n_m: int = 16,
               psi_hidden=(32, 32), phi_hidden=(64, 64), normalization=None,
               out_scale: float = 1.0) -> GnnModel:
    """Random-init model; psi drawn before phi as in ``gnn.py:87-104``."""
    nx = 2 * n_p
    psi = mlp_init([nx, *psi_hidden, n_m], rng)
    phi = mlp_init([nx + n_m + n_u, *phi_hidden, n_p], rng, out_scale=out_scale)
    nrm = normalization or Normalization.identity(nx, n_u)
    return GnnModel(psi=psi, phi=phi, dt=dt, n_p=n_p, n_u=n_u, n_m=n_m, normalization=nrm)


# ---------------------------------------------------------------------------
# forward model (device)
# ---------------------------------------------------------------------------

def step_array(model, topo, X, U) -> np.ndarray:
    """One dynamics step, batched over leading axes (``gnn.py:153-159``)."""
    X = np.asarray(X, dtype=float)
    U = np.asarray(U, dtype=float)
    lead = X.shape[:-2]
    M, nx = X.shape[-2:]
    if U.shape[:-1] != lead:
        U = np.broadcast_to(U, lead + U.shape[-1:])
    P = int(np.prod(lead)) if lead else 1
    eng = _dev.engine(topo, model)
    Xd = eng.h2d(X.reshape(P, M, nx), np.float64)
    Ud = eng.h2d(np.ascontiguousarray(U).reshape(P, -1), np.float64)
    f = eng.empty((P, M, nx), np.float64)
    eng.ctx.call("gm_step", P, Xd.data_ptr(), Ud.data_ptr(), f.data_ptr(), eng.stream_ptr())
    return f.cpu().numpy().reshape(X.shape)


def gnn_step(model, topo, x: SystemState, u: InputVector) -> SystemState:
    if x.node_count != topo.node_count:
        raise ValueError("state node count does not match topology")
    if x.array.shape[1] != model.n_state:
        raise ValueError("node state dimension does not match model")
    if u.n_u != model.n_u:
        raise ValueError("input dimension does not match model")
    return SystemState(step_array(model, topo, x.array, u.u))


def rollout(model, topo, x0: SystemState, inputs) -> Trajectory:
    """Open-loop prediction (``gnn.py:173-182``); each step runs on the GPU."""
    U = np.stack([u.u if isinstance(u, InputVector) else np.asarray(u, float) for u in inputs]) \
        if len(inputs) else np.zeros((0,))
    if U.shape[0] == 0:
        raise ValueError("inputs must be non-empty")
    eng = _dev.engine(topo, model)
    M, nx = x0.array.shape
    states = eng.empty((U.shape[0] + 1, M, nx), np.float64)
    states[0].copy_(eng.h2d(x0.array, np.float64))
    Ud = eng.h2d(U, np.float64)
    for k in range(U.shape[0]):
        eng.ctx.call("gm_step", 1, states[k].data_ptr(), Ud[k].data_ptr(), states[k + 1].data_ptr(),
                     eng.stream_ptr())
    return Trajectory(states=states.cpu().numpy(), inputs=U, dt=model.dt)


# ---------------------------------------------------------------------------
# linearisation
# ---------------------------------------------------------------------------

class LinearizedDynamics:
    """Per-stage, per-node affine blocks (``gnn.py:185-234``).

    x_i[k+1] = A_self[k,i] x_i[k] + sum_e A_nbr[k,e] x_src(e)[k] + B[k,i] u[k] + c[k,i]

    Constructed either from NumPy arrays (reference style; uploaded on use) or
    by ``linearize_trajectory`` with device-resident fp32 blocks, in which case
    ``a_self`` / ``a_nbr`` / ``b`` / ``c`` are materialised (fp64, read-only)
    on first access.
    """

    _FIELDS = ("a_self", "a_nbr", "b", "c")

    def __init__(self, topology, horizon, a_self=None, a_nbr=None, b=None, c=None, *, _device=None):
        self.topology = topology
        self.horizon = int(horizon)
        self._device = _device  # dict of fp32 torch tensors or None
        self._host = {}
        if _device is None:
            for name, arr in zip(self._FIELDS, (a_self, a_nbr, b, c)):
                self._host[name] = np.asarray(arr, dtype=float)
            self._validate()
        else:
            self._shapes = {k: tuple(v.shape) for k, v in _device.items()}

    def _validate(self):
        M = self.topology.node_count
        E = len(self.topology.edges)
        N = self.horizon
        a_self, a_nbr, b, c = (self._host[k] for k in self._FIELDS)
        nx = a_self.shape[-1]
        if a_self.shape != (N, M, nx, nx):
            raise ValueError("a_self shape mismatch")
        if a_nbr.shape[:2] != (N, E):
            raise ValueError("a_nbr shape mismatch")
        if b.shape[:2] != (N, M) or c.shape != (N, M, nx):
            raise ValueError("b/c shape mismatch")

    def _get(self, name):
        arr = self._host.get(name)
        if arr is None:
            arr = self._device[name].double().cpu().numpy()
            arr.flags.writeable = False
            self._host[name] = arr
        return arr

    a_self = property(lambda self: self._get("a_self"))
    a_nbr = property(lambda self: self._get("a_nbr"))
    b = property(lambda self: self._get("b"))
    c = property(lambda self: self._get("c"))

    def _shape(self, name):
        if self._device is not None:
            return self._shapes[name]
        return self._host[name].shape

    @property
    def n_state(self) -> int:
        return self._shape("a_self")[-1]

    @property
    def n_u(self) -> int:
        return self._shape("b")[-1]

    @property
    def on_device(self) -> bool:
        return self._device is not None

    def device_blocks(self, eng):
        """Device tensors (a_self, a_nbr, b fp32; c fp64) for engine ``eng``."""
        if self._device is not None and self._device["a_self"].device == eng.device:
            return tuple(self._device[k] for k in self._FIELDS)
        return tuple(eng.h2d(self._get(k), np.float64 if k == "c" else np.float32)
                     for k in self._FIELDS)

    def a_block(self, k: int, i: int, j: int) -> np.ndarray:
        if j == i:
            return self.a_self[k, i]
        for e, (di, sj) in enumerate(self.topology.edges):
            if di == i and sj == j:
                return self.a_nbr[k, e]
        raise KeyError(f"node {j} is not in the closed neighborhood of node {i}")

    def stage(self, k: int) -> "LinearizedDynamics":
        if self._device is not None:
            return LinearizedDynamics(self.topology, 1, _device={
                n: t[k : k + 1] for n, t in self._device.items()})
        return LinearizedDynamics(self.topology, 1, self.a_self[k : k + 1], self.a_nbr[k : k + 1],
                                  self.b[k : k + 1], self.c[k : k + 1])


def linearize_device(eng, X, U):
    """Run K-LIN on device tensors X (P, M, nx) fp64, U (P, nu) fp64;
    returns the four fp32 block tensors."""
    P, M, nx = X.shape
    E = eng.E
    nu = U.shape[-1]
    a_self = eng.empty((P, M, nx, nx), np.float32)
    a_nbr = eng.empty((P, E, nx, nx), np.float32)
    b = eng.empty((P, M, nx, nu), np.float32)
    c = eng.empty((P, M, nx), np.float64)
    eng.ctx.call("gm_linearize", P, X.data_ptr(), U.data_ptr(), a_self.data_ptr(),
                 a_nbr.data_ptr() if E else None, b.data_ptr(), c.data_ptr(), None,
                 eng.stream_ptr())
    return a_self, a_nbr, b, c


def _linearize(model, topo, X, U) -> LinearizedDynamics:
    X = np.asarray(X, dtype=float)
    U = np.asarray(U, dtype=float)
    eng = _dev.engine(topo, model)
    Xd = eng.h2d(X, np.float64)
    Ud = eng.h2d(U, np.float64)
    a_self, a_nbr, b, c = linearize_device(eng, Xd, Ud)
    return LinearizedDynamics(topo, X.shape[0],
                              _device=dict(a_self=a_self, a_nbr=a_nbr, b=b, c=c))


def linearize_stage(model, topo, x: SystemState, u: InputVector) -> LinearizedDynamics:
    """Jacobian blocks at a single point (``gnn.py:301-305``)."""
    return _linearize(model, topo, x.array[None], u.u[None])


def linearize_trajectory(model, topo, states, inputs) -> LinearizedDynamics:
    """Stage-wise linearisation along a nominal trajectory (``gnn.py:308-321``):
    states (N, M, nx) or (N+1, ...), of which the first N are used."""
    inputs = np.asarray(inputs, dtype=float)
    states = np.asarray(states, dtype=float)
    N = inputs.shape[0]
    if states.shape[0] not in (N, N + 1):
        raise ValueError("need one linearization state per stage")
    return _linearize(model, topo, states[:N], inputs)


# ---------------------------------------------------------------------------
# model file (gnn.py:324-378): JSON with dt, dims, normalization, weights
# ---------------------------------------------------------------------------

def save_model(model: GnnModel, path) -> None:
    def mlp_doc(m):
        return {"layer_dims": m.layer_dims, "weights": [W.tolist() for W in m.weights],
                "biases": [b.tolist() for b in m.biases]}

    nrm = model.normalization
    doc = {"dt": model.dt, "dims": {"n_p": model.n_p, "n_u": model.n_u, "n_m": model.n_m},
           "normalization": {"state_mean": nrm.state_mean.tolist(),
                             "state_scale": nrm.state_scale.tolist(),
                             "input_mean": nrm.input_mean.tolist(),
                             "input_scale": nrm.input_scale.tolist()},
           "psi": mlp_doc(model.psi), "phi": mlp_doc(model.phi)}
    with open(path, "w") as f:
        json.dump(doc, f)


def load_model(path) -> GnnModel:
    with open(path) as f:
        doc = json.load(f)
    try:
        dims, nrm = doc["dims"], doc["normalization"]

        def mlp(key):
            d = doc[key]
            return MlpParams(d["layer_dims"], [np.array(W, dtype=float) for W in d["weights"]],
                             [np.array(b, dtype=float) for b in d["biases"]])

        return GnnModel(psi=mlp("psi"), phi=mlp("phi"), dt=float(doc["dt"]), n_p=int(dims["n_p"]),
                        n_u=int(dims["n_u"]), n_m=int(dims["n_m"]),
                        normalization=Normalization(nrm["state_mean"], nrm["state_scale"],
                                                    nrm["input_mean"], nrm["input_scale"]))
    except (KeyError, TypeError) as exc:
        raise ValueError(f"malformed model file {path}: {exc}") from exc
