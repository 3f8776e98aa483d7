"""Receding-horizon control on the GPU -- reference-compatible API.

Mirrors ``gnnmpc/mpc.py``: ``MpcConfig`` (``:26-48``), ``StepTiming``
(``:51-56``), ``MpcState`` (``:59-72``), ``mpc_init`` (``:75-79``),
``mpc_step`` (``:102-200``), ``run_closed_loop`` (``:224-264``),
``ClosedLoopLog`` / ``write_closed_loop_csv``.  ``model`` may be a GnnModel
(linearised by K-LIN) or any ``Linearizer`` callable
``(states, inputs) -> LinearizedDynamics`` (the reference's plugin point,
``mpc.py:23``, ``:82-87``); its blocks are uploaded and the rest of the step
runs on the device.

One RTI step is a fixed chain of sm_100a kernels on one stream with no host
synchronisation until the single small read of ``[u_applied, status,
iterations]`` at the end:

    K-LIN -> K-REC (N stages) -> K-HG -> K-CON -> soft expansion -> K-QP -> K-RS

The controller state (``MpcState``) stays device-resident between steps; its
NumPy views are materialised lazily when a caller reads them.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import device as _dev
from ._runtime import lib
from .condensing import cost_device, rows_device, spec_rows
from .gnn import LinearizedDynamics, linearize_device
from .graph import InputVector, SystemState, Trajectory
from .qpsolver import STATUS_BY_CODE, QpStatus, SolverSettings


@dataclass
class MpcConfig:
    horizon: int
    dt: float
    solver: SolverSettings = field(default_factory=SolverSettings)
    warm_start: bool = True
    fallback: str = "hold-previous-input"
    sqp_iterations: int = 1
    sqp_damping: float = 1.0
    threads: int = 1
    input_filter_tau: float | None = None

    def __post_init__(self):
        if self.horizon < 1:
            raise ValueError("horizon must be >= 1")
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.fallback not in ("hold-previous-input", "zero-input"):
            raise ValueError("unknown fallback policy")
        if self.sqp_iterations < 1:
            raise ValueError("sqp_iterations must be >= 1")
        if not 0.0 < self.sqp_damping <= 1.0:
            raise ValueError("sqp_damping must be in (0, 1]")


@dataclass
class StepTiming:
    linearize_ms: float = 0.0
    condense_ms: float = 0.0
    solve_ms: float = 0.0
    total_ms: float = 0.0


class MpcState:
    """Linearisation trajectory plus bookkeeping (``mpc.py:59-72``).

    Array fields may be NumPy arrays (reference style) or device tensors
    (what ``mpc_step`` returns); reading an attribute always yields NumPy."""

    _ARRAYS = ("lin_states", "lin_inputs", "last_applied", "planned_states", "planned_inputs",
               "filtered_input")

    def __init__(self, lin_states, lin_inputs, step_count=0, last_applied=None,
                 planned_states=None, planned_inputs=None, last_status=None, last_iterations=0,
                 last_timing=None, filtered_input=None):
        self._vals = {}
        self.lin_states = lin_states
        self.lin_inputs = lin_inputs
        self.last_applied = last_applied
        self.planned_states = planned_states
        self.planned_inputs = planned_inputs
        self.filtered_input = filtered_input
        self.step_count = step_count
        self.last_status = last_status
        self.last_iterations = last_iterations
        self.last_timing = last_timing if last_timing is not None else StepTiming()

    def __getattr__(self, name):
        if name in MpcState._ARRAYS:
            v = self.__dict__["_vals"].get(name)
            if v is not None and not isinstance(v, np.ndarray):
                v = v.cpu().numpy()
                self.__dict__["_vals"][name] = v
            return v
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in MpcState._ARRAYS:
            self.__dict__.setdefault("_vals", {})[name] = value
        else:
            object.__setattr__(self, name, value)

    def device_value(self, name):
        """Raw stored value (tensor or ndarray) without materialising."""
        return self._vals.get(name)


def mpc_init(x_measured: SystemState, cfg: MpcConfig, n_u: int) -> MpcState:
    """All linearisation states at the measurement, inputs zero (``mpc.py:75-79``)."""
    N = cfg.horizon
    return MpcState(lin_states=np.tile(x_measured.array, (N + 1, 1, 1)),
                    lin_inputs=np.zeros((N, n_u)))


def _is_gnn_model(model) -> bool:
    return all(hasattr(model, a) for a in ("psi", "phi", "dt", "n_p", "n_u", "n_m",
                                           "normalization"))


class _Workspace:
    """Device buffers reused across steps for one (engine, N, constraint layout)."""

    def __init__(self, eng, N, nx, nu, rows):
        self.N, self.nx, self.nu = N, nx, nu
        M, E = eng.M, eng.E
        self.ld = lib().gm_gamma_ld(N, nu)
        self.n0 = N * nu
        self.m0 = rows.m0
        self.soft_idx = rows.soft_idx
        self.ns = int(self.soft_idx.size)
        self.n = self.n0 + self.ns
        self.m = self.m0 + self.ns
        f32, f64, i32 = np.float32, np.float64, np.int32
        self.a_self = eng.empty((N, M, nx, nx), f32)
        self.a_nbr = eng.empty((N, E, nx, nx), f32)
        self.b = eng.empty((N, M, nx, nu), f32)
        self.c = eng.empty((N, M, nx), f64)
        self.W = eng.empty((M, N + 1, nx, self.ld), f32)
        self.H0 = eng.empty((self.n0, self.n0), f64)
        self.g0 = eng.empty((self.n0,), f64)
        self.C0 = eng.empty((self.m0, self.n0), f64)
        self.d0 = eng.empty((self.m0,), f64)
        if self.ns:
            self.H = eng.empty((self.n, self.n), f64)
            self.g = eng.empty((self.n,), f64)
            self.C = eng.empty((self.m, self.n), f64)
            self.d = eng.empty((self.m,), f64)
            self.idx = eng.h2d(self.soft_idx, i32)
        else:
            self.H, self.g, self.C, self.d = self.H0, self.g0, self.C0, self.d0
        self.warm = eng.zeros((self.n,), f64)
        self.u = eng.empty((self.n,), f64)
        self.lam = eng.empty((max(self.m, 1),), f64)
        self.status = eng.empty((1,), i32)
        self.iters = eng.empty((1,), i32)
        self.resid = eng.empty((1, 3), f64)
        self.summary = eng.empty((nu + 2,), f64)
        self.host_summary = eng.torch.empty((nu + 2,), dtype=eng.torch.float64, pin_memory=True)
        self.events = [eng.torch.cuda.Event(enable_timing=True) for _ in range(4)]


def _workspace(eng, N, nx, nu, rows):
    key = ("ws", N, nx, nu, rows.m0, tuple(rows.soft_idx.tolist()))
    ws = eng.cache.get(key)
    if ws is None:
        ws = _Workspace(eng, N, nx, nu, rows)
        eng.cache[key] = ws
    return ws


def _as_device(eng, value, shape, dtype=np.float64):
    if value is None:
        return None
    if isinstance(value, np.ndarray) or not hasattr(value, "data_ptr"):
        return eng.h2d(np.asarray(value, dtype=float).reshape(shape), dtype)
    return value


def mpc_step(model, topo, spec, x_measured: SystemState, state: MpcState, cfg: MpcConfig):
    """One control step of the receding-horizon loop (``mpc.py:102-200``).

    Returns the applied ``InputVector`` and the successor ``MpcState`` whose
    linearisation trajectory is the one-step-shifted plan."""
    t_start = time.perf_counter()
    torch = _dev.require_cuda() if hasattr(_dev, "require_cuda") else None
    N = cfg.horizon
    gnn = _is_gnn_model(model)
    if not gnn and not callable(model):
        raise TypeError("model must be a GnnModel or a linearizer callable")
    eng = _dev.engine(topo, model if gnn else None)
    torch = eng.torch
    M = topo.node_count
    lin_in_prev = state.device_value("lin_inputs")
    n_u = int(lin_in_prev.shape[1])
    nx = int(np.asarray(x_measured.array).shape[1])
    eng.set_dims(nx, n_u)
    rows = spec_rows(spec, nx, n_u)
    ws = _workspace(eng, N, nx, n_u, rows)
    sp = eng.stream_ptr()
    ev = ws.events
    stream = torch.cuda.current_stream(eng.device)

    # trajectory with the measurement at stage 0 (mpc.py:120-122)
    x_meas = eng.h2d(x_measured.array, np.float64)
    fb_states = torch.empty((N + 1, M, nx), dtype=torch.float64, device=eng.device)
    fb_states.copy_(_as_device(eng, state.device_value("lin_states"), (N + 1, M, nx)))
    fb_states[0].copy_(x_meas)
    fb_inputs = _as_device(eng, lin_in_prev, (N, n_u)).clone()
    ls, li = fb_states, fb_inputs
    prev = state.device_value("last_applied")
    u_prev = _as_device(eng, prev, (n_u,)) if prev is not None else None

    cur = torch.empty_like(fb_states) if cfg.sqp_iterations > 1 else None
    planned_states = torch.empty((M, N + 1, nx), dtype=torch.float64, device=eng.device)
    planned_inputs = torch.empty((N, n_u), dtype=torch.float64, device=eng.device)
    next_states = torch.empty((N + 1, M, nx), dtype=torch.float64, device=eng.device)
    next_inputs = torch.empty((N, n_u), dtype=torch.float64, device=eng.device)
    u_applied = torch.empty((n_u,), dtype=torch.float64, device=eng.device)

    timing = StepTiming()
    total_iters = 0
    status_code = None
    for it in range(cfg.sqp_iterations):
        ev[0].record(stream)
        # stage 1: linearise along the first N states (mpc.py:130-132)
        if gnn:
            if not ls.is_contiguous():
                ls = ls.contiguous()
            a_self, a_nbr, b, c = ws.a_self, ws.a_nbr, ws.b, ws.c
            eng.ctx.call("gm_linearize", N, ls.data_ptr(), li.data_ptr(), a_self.data_ptr(),
                         a_nbr.data_ptr() if eng.E else None, b.data_ptr(), c.data_ptr(), None, sp)
        else:
            lin = model(ls[:N].cpu().numpy(), li.cpu().numpy())
            a_self, a_nbr, b, c = lin.device_blocks(eng) if isinstance(lin, LinearizedDynamics) \
                else tuple(eng.h2d(getattr(lin, k), np.float64 if k == "c" else np.float32)
                           for k in ("a_self", "a_nbr", "b", "c"))
        ev[1].record(stream)
        # stage 2-3: condensing (mpc.py:135-137)
        eng.ctx.call("gm_condense_gammas", 1, N, a_self.data_ptr(),
                     a_nbr.data_ptr() if eng.E else None, b.data_ptr(), c.data_ptr(),
                     x_meas.data_ptr(), ws.W.data_ptr(), ws.ld, sp)
        cost_device(eng, spec, ws.W, ws.ld, N, nx, n_u, ws.H0, ws.g0)
        rows_device(eng, rows, ws.W, ws.ld, N, ws.C0, ws.d0)
        if ws.ns:
            r1 = eng.h2d(rows.rho1[ws.soft_idx], np.float64)
            r2 = eng.h2d(rows.rho2[ws.soft_idx], np.float64)
            eng.ctx.call("gm_expand_soft", 1, ws.n0, ws.m0, ws.H0.data_ptr(), ws.g0.data_ptr(),
                         ws.C0.data_ptr(), ws.d0.data_ptr(), ws.ns, ws.idx.data_ptr(),
                         r1.data_ptr(), r2.data_ptr(), ws.H.data_ptr(), ws.g.data_ptr(),
                         ws.C.data_ptr(), ws.d.data_ptr(), sp)
        ev[2].record(stream)
        # stage 4: QP with warm start [lin_inputs; 0] (mpc.py:140-147)
        warm = None
        if cfg.warm_start:
            ws.warm[: N * n_u].copy_(li.reshape(-1))
            warm = ws.warm.data_ptr()
        cs = cfg.solver.as_c()
        import ctypes

        eng.ctx.call("gm_solve_qp", 1, ws.n, ws.m, ws.H.data_ptr(), ws.g.data_ptr(),
                     ws.C.data_ptr() if ws.m else None, ws.d.data_ptr() if ws.m else None, warm,
                     ctypes.byref(cs), ws.u.data_ptr(), ws.lam.data_ptr(), ws.status.data_ptr(),
                     ws.iters.data_ptr(), ws.resid.data_ptr(), sp)
        ev[3].record(stream)
        # RTI epilogue on the device (mpc.py:151-200)
        eng.ctx.call("gm_mpc_finish", 1, N, ws.W.data_ptr(), ws.ld, ws.u.data_ptr(), ws.n,
                     ws.status.data_ptr(), ws.iters.data_ptr(), ls.data_ptr(), li.data_ptr(),
                     fb_states.data_ptr(), fb_inputs.data_ptr(), float(cfg.sqp_damping),
                     0 if cfg.fallback == "hold-previous-input" else 1,
                     u_prev.data_ptr() if u_prev is not None else None, int(u_prev is not None),
                     cur.data_ptr() if cur is not None else None, planned_states.data_ptr(),
                     planned_inputs.data_ptr(), next_states.data_ptr(), next_inputs.data_ptr(),
                     u_applied.data_ptr(), ws.summary.data_ptr(), sp)
        ws.host_summary.copy_(ws.summary, non_blocking=True)
        stream.synchronize()
        summ = ws.host_summary.numpy()
        status_code = int(summ[n_u])
        total_iters += int(summ[n_u + 1])
        timing.linearize_ms += ev[0].elapsed_time(ev[1])
        timing.condense_ms += ev[1].elapsed_time(ev[2])
        timing.solve_ms += ev[2].elapsed_time(ev[3])
        if status_code > 1:  # not OPTIMAL / MAX_ITERATIONS: fallback already applied
            break
        if it + 1 < cfg.sqp_iterations:
            ls, li = cur.clone(), planned_inputs.clone()

    u_app = summ[:n_u].copy()
    filtered = state.device_value("filtered_input")
    if cfg.input_filter_tau is not None:  # optional first-order smoothing (mpc.py:178-183)
        alpha = cfg.dt / (cfg.input_filter_tau + cfg.dt)
        prevf = np.asarray(filtered.cpu().numpy() if hasattr(filtered, "cpu") else filtered,
                           dtype=float) if filtered is not None else u_app
        u_app = prevf + alpha * (u_app - prevf)
        filtered = u_app.copy()
        last_applied = u_app.copy()
    else:
        last_applied = u_applied
    timing.total_ms = (time.perf_counter() - t_start) * 1e3
    new_state = MpcState(lin_states=next_states, lin_inputs=next_inputs,
                         step_count=state.step_count + 1, last_applied=last_applied,
                         planned_states=planned_states, planned_inputs=planned_inputs,
                         last_status=STATUS_BY_CODE[status_code], last_iterations=total_iters,
                         last_timing=timing, filtered_input=filtered)
    return InputVector(u_app), new_state


@dataclass
class ClosedLoopLog:
    states: np.ndarray
    inputs: np.ndarray
    statuses: list
    iterations: np.ndarray
    timings: np.ndarray
    node_errors: np.ndarray
    dt: float

    @property
    def n_steps(self) -> int:
        return self.inputs.shape[0]

    def optimal_fraction(self) -> float:
        return sum(1 for s in self.statuses if s == QpStatus.OPTIMAL) / max(1, len(self.statuses))

    def to_trajectory(self) -> Trajectory:
        return Trajectory(states=self.states, inputs=self.inputs, dt=self.dt)


def run_closed_loop(plant_step, model, topo, spec_provider, x0: SystemState, n_steps: int,
                    cfg: MpcConfig) -> ClosedLoopLog:
    """Alternate controller and plant (``mpc.py:224-264``)."""
    n_u = spec_provider(0, None).n_u if callable(spec_provider) else spec_provider.n_u
    state = mpc_init(x0, cfg, n_u)
    M = x0.node_count
    states = np.empty((n_steps + 1, M, x0.array.shape[1]))
    states[0] = x0.array
    inputs = np.empty((n_steps, n_u))
    statuses = []
    iterations = np.zeros(n_steps, dtype=int)
    timings = np.zeros((n_steps, 4))
    node_errors = np.zeros((n_steps, M))
    x = x0
    for t in range(n_steps):
        spec = spec_provider(t, state) if callable(spec_provider) else spec_provider
        u, state = mpc_step(model, topo, spec, x, state, cfg)
        n_p = x.n_p
        node_errors[t] = np.linalg.norm(x.positions - spec.x_ref[:, 0, :n_p], axis=1)
        inputs[t] = u.u
        statuses.append(state.last_status)
        iterations[t] = state.last_iterations
        tm = state.last_timing
        timings[t] = (tm.linearize_ms, tm.condense_ms, tm.solve_ms, tm.total_ms)
        x = plant_step(x, u)
        states[t + 1] = x.array
    return ClosedLoopLog(states, inputs, statuses, iterations, timings, node_errors, cfg.dt)


def write_closed_loop_csv(path, log: ClosedLoopLog) -> None:
    n_u = log.inputs.shape[1]
    M = log.node_errors.shape[1]
    header = (["step", "t", "status", "iters", "linearize_ms", "condense_ms", "solve_ms",
               "total_ms"] + [f"u_{i+1}" for i in range(n_u)] + [f"err_node_{i+1}" for i in range(M)])
    with open(path, "w") as f:
        f.write(",".join(header) + "\n")
        for k in range(log.n_steps):
            row = [str(k), "%.17g" % (k * log.dt), log.statuses[k].value, str(int(log.iterations[k]))]
            row += ["%.17g" % v for v in log.timings[k]]
            row += ["%.17g" % v for v in log.inputs[k]]
            row += ["%.17g" % v for v in log.node_errors[k]]
            f.write(",".join(row) + "\n")
