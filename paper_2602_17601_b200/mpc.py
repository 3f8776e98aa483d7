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
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import device as _dev
from ._runtime import lib
from .condensing import fused_device, lin_blocks, rows_device
from .gnn import LinearizedDynamics, linearize_device
from .graph import InputVector, SystemState, Trajectory
from .qpsolver import STATUS_BY_CODE, QpStatus, SolverSettings, settings_c


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


def _field(state, name):
    """Raw value of an MpcState field for ours (device tensors kept) or the
    reference's NumPy dataclass."""
    if hasattr(state, "device_value"):
        return state.device_value(name)
    return getattr(state, name, None)


def _is_gnn_model(model) -> bool:
    return all(hasattr(model, a) for a in ("psi", "phi", "dt", "n_p", "n_u", "n_m",
                                           "normalization"))


class StepPlan:
    """Device buffers and the kernel chain of one RTI step for a fixed
    (engine, spec, horizon, config).  ``enqueue`` issues

        K-LIN -> K-REC -> K-HG -> K-CON -> soft expansion -> K-QP -> K-RS

    on the current stream with no host synchronisation and no host->device
    copies; every input it reads lives in the plan's static buffers, so the
    three stage groups can be captured once as CUDA graphs and replayed."""

    def __init__(self, eng, ds, N, nx, nu, cfg, gnn):
        torch = eng.torch
        self.eng, self.ds, self.N, self.nx, self.nu, self.gnn = eng, ds, N, nx, nu, gnn
        self.cfg = cfg
        M, E = eng.M, eng.E
        self.M = M
        self.ld = lib().gm_gamma_ld(N, nu)
        self.n0 = N * nu
        self.m0 = ds.rows.m0
        self.ns = ds.ns
        self.n = self.n0 + self.ns
        self.m = self.m0 + self.ns
        f32, f64, i32 = np.float32, np.float64, np.int32
        e = eng.empty
        # static inputs
        self.x_meas = e((M, nx), f64)
        # [lin_states | lin_inputs | u_prev] in one buffer, laid out like the
        # tail [next_states | next_inputs | u_applied] of the output snapshot,
        # so a state this function returned comes back in with one copy
        a, b = (N + 1) * M * nx, N * nu
        self.inbuf = eng.zeros((a + b + nu,), f64)
        self.ls = self.inbuf[:a].view(N + 1, M, nx)  # linearisation trajectory, [0] = x_measured
        self.li = self.inbuf[a:a + b].view(N, nu)
        self.fb_states = self.ls            # RTI: fallback plan == input plan
        self.fb_inputs = self.li
        self.u_prev = self.inbuf[a + b:]    # zeros == "no previous input" (mpc.py:413)
        # scratch
        self.a_self = e((N, M, nx, nx), f32)
        self.a_nbr = e((N, max(E, 1), nx, nx), f32)
        self.b = e((N, M, nx, nu), f32)
        self.c = e((N, M, nx), f64)
        self.W = e((M, N + 1, nx, self.ld), f32)
        self.H0 = e((self.n0, self.n0), f64)
        self.g0 = e((self.n0,), f64)
        self.C0 = e((max(self.m0, 1), self.n0), f64)
        self.d0 = e((max(self.m0, 1),), f64)
        if self.ns:
            self.H = e((self.n, self.n), f64)
            self.g = e((self.n,), f64)
            self.C = e((self.m, self.n), f64)
            self.d = e((self.m,), f64)
        else:
            self.H, self.g, self.C, self.d = self.H0, self.g0, self.C0, self.d0
        self.warm = eng.zeros((self.n,), f64)
        self.u = e((self.n,), f64)
        self.lam = e((max(self.m, 1),), f64)
        self.status = e((1,), i32)
        self.iters = e((1,), i32)
        self.resid = e((1, 3), f64)
        # static outputs; the four arrays a new MpcState keeps live in one
        # buffer so the state is snapshotted with a single device copy
        self.cur = e((N + 1, M, nx), f64)
        sizes = [M * (N + 1) * nx, N * nu, (N + 1) * M * nx, N * nu, nu]
        self.outbuf = e((sum(sizes),), f64)
        self.in_off = sizes[0] + sizes[1]   # where [next_states | next_inputs | u_applied] starts
        self.out_views = self._carve(self.outbuf)
        (self.planned_states, self.planned_inputs, self.next_states, self.next_inputs,
         self.u_applied) = self.out_views
        self.summary = e((nu + 2,), f64)
        self.host_summary = torch.empty((nu + 2,), dtype=torch.float64, pin_memory=True)
        self.host_x = torch.empty((M, nx), dtype=torch.float64, pin_memory=True)
        # external timing events: recorded as event nodes inside the step graph
        self.events = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
        self._ev_handles = None
        self.graphs = None
        self.graph = None
        self.settings_c = settings_c(cfg.solver)

    def _carve(self, buf):
        M, N, nx, nu = self.M, self.N, self.nx, self.nu
        sizes = [M * (N + 1) * nx, N * nu, (N + 1) * M * nx, N * nu, nu]
        shapes = [(M, N + 1, nx), (N, nu), (N + 1, M, nx), (N, nu), (nu,)]
        out, o = [], 0
        for sz, sh in zip(sizes, shapes):
            out.append(buf[o:o + sz].view(sh))
            o += sz
        return out

    # -- the three stage groups ------------------------------------------------
    def _linearize(self):
        eng, N = self.eng, self.N
        eng.ctx.call("gm_linearize", N, self.ls.data_ptr(), self.li.data_ptr(),
                     self.a_self.data_ptr(), self.a_nbr.data_ptr() if eng.E else None,
                     self.b.data_ptr(), self.c.data_ptr(), None, eng.stream_ptr())

    def _condense(self):
        eng, N, ds = self.eng, self.N, self.ds
        sp = eng.stream_ptr()
        fused_device(eng, ds, self.a_self, self.a_nbr if eng.E else None, self.b, self.c,
                     self.x_meas, self.W, self.ld, N, self.H0, self.g0)
        rows_device(eng, ds, self.W, self.ld, N, self.C0, self.d0)
        if self.ns:
            eng.ctx.call("gm_expand_soft", 1, self.n0, self.m0, self.H0.data_ptr(),
                         self.g0.data_ptr(), self.C0.data_ptr(), self.d0.data_ptr(), self.ns,
                         ds.idx.data_ptr(), ds.rho1.data_ptr(), ds.rho2.data_ptr(),
                         self.H.data_ptr(), self.g.data_ptr(), self.C.data_ptr(),
                         self.d.data_ptr(), sp)

    def _solve_finish(self):
        import ctypes

        eng, N, cfg = self.eng, self.N, self.cfg
        sp = eng.stream_ptr()
        warm = None
        if cfg.warm_start:  # warm start [lin_inputs; 0] (mpc.py:384-388)
            self.warm[: N * self.nu].copy_(self.li.reshape(-1))
            warm = self.warm.data_ptr()
        eng.ctx.call("gm_solve_qp", 1, self.n, self.m, self.H.data_ptr(), self.g.data_ptr(),
                     self.C.data_ptr() if self.m else None, self.d.data_ptr() if self.m else None,
                     warm, ctypes.byref(self.settings_c), self.u.data_ptr(), self.lam.data_ptr(),
                     self.status.data_ptr(), self.iters.data_ptr(), self.resid.data_ptr(), sp)
        eng.ctx.call("gm_mpc_finish", 1, N, self.W.data_ptr(), self.ld, self.u.data_ptr(), self.n,
                     self.status.data_ptr(), self.iters.data_ptr(), self.ls.data_ptr(),
                     self.li.data_ptr(), self.fb_states.data_ptr(), self.fb_inputs.data_ptr(),
                     float(cfg.sqp_damping), 0 if cfg.fallback == "hold-previous-input" else 1,
                     self.u_prev.data_ptr(), 1, self.cur.data_ptr(),
                     self.planned_states.data_ptr(), self.planned_inputs.data_ptr(),
                     self.next_states.data_ptr(), self.next_inputs.data_ptr(),
                     self.u_applied.data_ptr(), self.summary.data_ptr(), sp)

    def groups(self):
        return (self._linearize, self._condense, self._solve_finish) if self.gnn \
            else (self._condense, self._solve_finish)

    def capture(self):
        """Record the whole step as one CUDA graph (after one eager run):
        measurement H2D from the pinned staging buffer, stage 0 of the
        linearisation trajectory, the three stage groups bracketed by timing
        event nodes, and the D2H of [u_applied, status, iterations] into
        pinned memory -- one launch per control step.  The per-group graphs
        are kept for eager-style replays (bench stage timing, launch counts)."""
        torch = self.eng.torch
        graphs = []
        for fn in self.groups():
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs.append(g)
        self.graphs = graphs
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.x_meas.copy_(self.host_x, non_blocking=True)
            self.ls[0].copy_(self.x_meas)
            self._issue(self.groups(), eager=True, timed=True)
            self.host_summary.copy_(self.summary, non_blocking=True)
        self.graph = g

    def _issue(self, groups, eager, timed):
        torch = self.eng.torch
        stream = torch.cuda.current_stream(self.eng.device)
        ev = self.events
        marks = [1, 2, 3] if len(groups) == 3 else [2, 3]
        if timed:
            ev[0].record(stream)
            if len(groups) == 2:
                ev[1].record(stream)
        for g, mark in zip(groups, marks):
            if eager:
                g()
            else:
                g.replay()
            if timed:
                ev[mark].record(stream)

    def enqueue(self, timed=True):
        """Issue the kernel chain of one step on the current stream (per-group
        graph replay if captured, else eager).  Events bracket linearize |
        condense | solve+epilogue for StepTiming."""
        if self.graphs is not None:
            self._issue(self.graphs, eager=False, timed=timed)
        else:
            self._issue(self.groups(), eager=True, timed=timed)

    def stage_ms(self):
        """(linearize, condense, solve) ms of the last run: one C call for the
        three event pairs (gm_event_times)."""
        import ctypes

        if self._ev_handles is None:
            self._ev_handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in self.events])
            self._ev_out = (ctypes.c_float * 3)()
        rc = lib().gm_event_times(4, ctypes.addressof(self._ev_handles), ctypes.addressof(self._ev_out))
        if rc != 0:
            ev = self.events
            return ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
        o = self._ev_out
        return float(o[0]), float(o[1]), float(o[2])


_MAX_PLANS = 16


def get_plan(eng, spec, N, nx, nu, cfg, gnn) -> StepPlan:
    from .condensing import device_spec

    ds = device_spec(eng, spec, nx, nu)
    s = cfg.solver
    # replayable: frozen specs, and tracking specs whose only moving part
    # (x_ref) is refreshed in place in the plan's device spec; their plans are
    # keyed by the cached device spec.  Specs rebuilt on every call (not
    # frozen, e.g. with moving constraint rows) share one eagerly enqueued plan
    # per row layout, re-pointed at the new device spec (no per-call buffers)
    replay = getattr(spec, "_frozen", False) or getattr(spec, "_static_token", None) is not None
    ident = id(ds) if replay else ("rows", ds.rows.m0, ds.ns)
    key = ("plan", ident, N, nx, nu, gnn, bool(cfg.warm_start), float(cfg.sqp_damping),
           cfg.fallback, float(s.tolerance), int(s.max_iterations), float(s.regularization),
           float(s.fraction_to_boundary))
    plan = eng.cache.get(key)
    if plan is not None and not replay:
        plan.ds = ds
    if plan is None or plan.ds is not ds:
        plan = StepPlan(eng, ds, N, nx, nu, cfg, gnn)
        plan.use_graphs = replay
        plan.runs = 0
        eng.cache[key] = plan
        if replay:
            # the plan lives as long as the spec (or the provider token) it
            # was built for: its buffers and graphs go when the owner goes
            owner = getattr(spec, "_static_token", None)
            weakref.finalize(owner if owner is not None else spec, eng.cache.pop, key, None)
        # bound the number of live plans per engine (each owns a Gamma array
        # and captured graphs): evict the oldest beyond _MAX_PLANS
        plans = [k for k in eng.cache if isinstance(k, tuple) and k and k[0] == "plan"]
        for k in plans[:-_MAX_PLANS]:
            eng.cache.pop(k, None)
    return plan


def _copy_in(dst, value, pinned=None):
    """Device copy of a state field (tensor -> D2D, ndarray -> H2D)."""
    if hasattr(value, "data_ptr") and not isinstance(value, np.ndarray):
        dst.copy_(value.reshape(dst.shape))
        return
    arr = np.asarray(value, dtype=float).reshape(tuple(dst.shape))
    if pinned is not None:
        pinned.numpy()[...] = arr
        dst.copy_(pinned, non_blocking=True)
    else:
        import torch

        dst.copy_(torch.from_numpy(np.ascontiguousarray(arr)))


def mpc_step(model, topo, spec, x_measured: SystemState, state: MpcState, cfg: MpcConfig):
    """One control step of the receding-horizon loop (``mpc.py:102-200``).

    Returns the applied ``InputVector`` and the successor ``MpcState`` whose
    linearisation trajectory is the one-step-shifted plan.  All stages run on
    the device; the only host<->device traffic is the measurement in, the
    (device-resident) previous plan, and one small read of
    [u_applied, status, iterations] out."""
    t_start = time.perf_counter()
    N = cfg.horizon
    gnn = _is_gnn_model(model)
    if not gnn and not callable(model):
        raise TypeError("model must be a GnnModel or a linearizer callable")
    eng = _dev.engine(topo, model if gnn else None)
    torch = eng.torch
    lin_in_prev = _field(state, "lin_inputs")
    n_u = int(lin_in_prev.shape[1])
    x_arr = x_measured.array
    x_on_device = hasattr(x_arr, "data_ptr") and not isinstance(x_arr, np.ndarray)
    nx = int(x_arr.shape[1])
    eng.set_dims(nx, n_u)
    plan = get_plan(eng, spec, N, nx, n_u, cfg, gnn)
    stream = torch.cuda.current_stream(eng.device)

    # inputs: measurement, previous plan with x_measured at stage 0 (mpc.py:120-122)
    graphable = plan.use_graphs and cfg.sqp_iterations == 1
    # the whole-step graph reads the measurement from the pinned host buffer;
    # a device-resident measurement goes through the per-group graphs
    whole = graphable and plan.graph is not None and not x_on_device
    # a state this plan returned: its trajectory, inputs and last applied input
    # are one contiguous piece of its snapshot -> one device copy
    snap = getattr(state, "_snapshot", None)
    fast = (snap is not None and snap[1] is plan and _field(state, "lin_states") is snap[2]
            and lin_in_prev is snap[3] and _field(state, "last_applied") is snap[4])
    if whole:  # the step graph does the H2D from the pinned buffer and ls[0]
        plan.host_x.numpy()[...] = np.asarray(x_measured.array, dtype=float).reshape(plan.host_x.shape)
    else:
        _copy_in(plan.x_meas, x_measured.array, plan.host_x)
    if fast:
        plan.inbuf.copy_(snap[0][plan.in_off:])
    else:
        _copy_in(plan.ls, _field(state, "lin_states"))
        _copy_in(plan.li, lin_in_prev)
        prev = _field(state, "last_applied")
        if prev is None:
            plan.u_prev.zero_()
        else:
            _copy_in(plan.u_prev, prev)
    if not whole:
        plan.ls[0].copy_(plan.x_meas)

    timing = StepTiming()
    total_iters = 0
    if cfg.sqp_iterations > 1:  # the SQP loop keeps the original plan as the fallback
        plan.fb_states = plan.ls.clone()
        plan.fb_inputs = plan.li.clone()
    else:
        plan.fb_states, plan.fb_inputs = plan.ls, plan.li
    early = None
    for it in range(cfg.sqp_iterations):
        if not gnn:  # plug-in Linearizer (mpc.py:23, :82-87): upload its blocks
            lin = model(plan.ls[:N].cpu().numpy(), plan.li.cpu().numpy())
            blocks = lin_blocks(lin, eng)
            for dst, src in zip((plan.a_self, plan.a_nbr, plan.b, plan.c), blocks):
                if src.numel():
                    dst.view(-1)[: src.numel()].copy_(src.reshape(-1))
        if whole:
            plan.graph.replay()
            if cfg.sqp_iterations == 1:
                # the snapshot copy and its views are enqueued / built while
                # the step runs (nothing writes outbuf after the graph)
                early = plan.outbuf.clone()
                early_views = plan._carve(early)
        else:
            if graphable and plan.graph is None and plan.runs >= 1:
                # make sure the eager copies of this call are done before the
                # capture's own side-stream work, then capture for later calls
                plan.capture()
            plan.enqueue()
            plan.host_summary.copy_(plan.summary, non_blocking=True)
        plan.runs += 1
        stream.synchronize()
        summ = plan.host_summary.numpy()
        status_code = int(summ[n_u])
        total_iters += int(summ[n_u + 1])
        lm, cm, sm = plan.stage_ms()
        timing.linearize_ms += lm if gnn else 0.0
        timing.condense_ms += cm
        timing.solve_ms += sm
        if status_code > 1:  # not OPTIMAL / MAX_ITERATIONS: fallback already applied
            break
        if it + 1 < cfg.sqp_iterations:
            plan.ls.copy_(plan.cur)
            plan.li.copy_(plan.planned_inputs)

    u_app = summ[:n_u].copy()
    filtered = _field(state, "filtered_input")
    if cfg.input_filter_tau is not None:  # optional first-order smoothing (mpc.py:178-183)
        alpha = cfg.dt / (cfg.input_filter_tau + cfg.dt)
        prevf = (np.asarray(filtered.cpu().numpy() if hasattr(filtered, "cpu") else filtered,
                            dtype=float) if filtered is not None else u_app)
        u_app = prevf + alpha * (u_app - prevf)
        filtered = u_app.copy()
        last_applied = u_app.copy()
    else:
        last_applied = None
    if early is not None:
        snap, views = early, early_views
    else:
        snap = plan.outbuf.clone()  # one device copy: the new state owns it
        views = plan._carve(snap)
    planned_states, planned_inputs, next_states, next_inputs, u_applied = views
    if last_applied is None:
        last_applied = u_applied
    new_state = MpcState(lin_states=next_states, lin_inputs=next_inputs,
                         step_count=state.step_count + 1, last_applied=last_applied,
                         planned_states=planned_states, planned_inputs=planned_inputs,
                         last_status=STATUS_BY_CODE[status_code], last_iterations=total_iters,
                         last_timing=timing, filtered_input=filtered)
    # private: lets the next call on this plan load [trajectory | inputs |
    # last input] with one copy (checked against the fields it then reads)
    object.__setattr__(new_state, "_snapshot", (snap, plan, next_states, next_inputs, u_applied))
    timing.total_ms = (time.perf_counter() - t_start) * 1e3
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
