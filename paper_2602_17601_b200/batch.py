"""Batched RTI steps over independent MPC instances (cfg4) and their sharding.

B instances (scenarios / robots) share one model, one topology and one
constraint layout; each has its own measurement, linearisation trajectory and
references.  Every stage is ONE launch over all instances -- the kernels take
an instance count (K-LIN: B*N linearisation points; K-REC / K-HG / K-CON /
soft expansion / K-QP / K-RS: B-strided arrays; K-QP runs one CTA per QP), so a
batch fills the GPU instead of looping over ``mpc_step``.

Sharding over GPUs (``shard_range``): instance b lives on rank b * world // B;
there is no data-path collective -- each rank steps its own shard.  The
reference has no batched or multi-device path; the
single-instance semantics are those of ``mpc_step`` (``mpc.py:102-200``) and
are checked instance by instance against the oracle in the tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import device as _dev
from ._runtime import lib
from .condensing import spec_rows
from .errors import ConfigurationError
from .mpc import MpcConfig
from .qpsolver import STATUS_BY_CODE, settings_c


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split of ``n_items`` over ``world`` ranks."""
    lo = (n_items * rank) // world
    hi = (n_items * (rank + 1)) // world
    return lo, hi


@dataclass
class BatchResult:
    u_applied: np.ndarray       # (B, nu)
    status: list                # QpStatus per instance
    iterations: np.ndarray      # (B,)
    next_states: object         # device (B, N+1, M, nx)
    next_inputs: object         # device (B, N, nu)


class BatchedMpc:
    """RTI controller for B independent instances on one device.

    ``spec`` provides the shared cost weights / constraints; per-instance
    references are passed as ``x_ref`` (B, M, N+1, nx) (the cfg4 recipe uses
    each instance's own initial state as its reference)."""

    def __init__(self, model, topo, spec, cfg: MpcConfig, B: int, device=None):
        if cfg.sqp_iterations != 1 or cfg.input_filter_tau is not None:
            # the batched step is the RTI step (one QP per instance per call);
            # the SQP loop and the input filter are per-instance host logic of
            # mpc_step (mpc.py:129-183) -- use mpc_step for those
            raise ConfigurationError("BatchedMpc supports sqp_iterations == 1 and no input filter")
        self.eng = eng = _dev.engine(topo, model, device)
        self.model, self.topo, self.spec, self.cfg, self.B = model, topo, spec, cfg, B
        torch = eng.torch
        N, nx, nu = cfg.horizon, 2 * model.n_p, model.n_u
        self.N, self.nx, self.nu = N, nx, nu
        eng.set_dims(nx, nu)
        M, E = eng.M, eng.E
        self.rows = rows = spec_rows(spec, nx, nu)
        self.ld = lib().gm_gamma_ld(N, nu)
        self.n0, self.m0 = N * nu, rows.m0
        self.soft_idx = rows.soft_idx
        self.ns = int(self.soft_idx.size)
        self.n, self.m = self.n0 + self.ns, self.m0 + self.ns
        f32, f64, i32 = np.float32, np.float64, np.int32
        e = eng.empty
        self.X = e((B, N + 1, M, nx), f64)
        self.U = e((B, N, nu), f64)
        self.x0 = e((B, M, nx), f64)
        self.xref = e((B, M, N + 1, nx), f64)
        self.q = eng.h2d(spec.q, f64)
        self.r = eng.h2d(spec.r, f64)
        self.uref = eng.h2d(spec.u_ref, f64)
        self.a_self = e((B, N, M, nx, nx), f32)
        self.a_nbr = e((B, N, max(E, 1), nx, nx), f32)
        self.b = e((B, N, M, nx, nu), f32)
        self.c = e((B, N, M, nx), f64)
        self.W = e((B * M, N + 1, nx, self.ld), f32)
        self.H0 = e((B, self.n0, self.n0), f64)
        self.g0 = e((B, self.n0), f64)
        self.C0 = e((B, max(self.m0, 1), self.n0), f64)
        self.d0 = e((B, max(self.m0, 1)), f64)
        if self.ns:
            self.H = e((B, self.n, self.n), f64)
            self.g = e((B, self.n), f64)
            self.C = e((B, self.m, self.n), f64)
            self.d = e((B, self.m), f64)
            self.idx = eng.h2d(self.soft_idx, i32)
            self.rho1 = eng.h2d(rows.rho1[self.soft_idx], f64)
            self.rho2 = eng.h2d(rows.rho2[self.soft_idx], f64)
        else:
            self.H, self.g, self.C, self.d = self.H0, self.g0, self.C0, self.d0
        self.dev_rows = [eng.h2d(a, dt) if a.size else None for a, dt in (
            (rows.in_stage, i32), (rows.in_c, f64), (rows.in_d, f64), (rows.st_node, i32),
            (rows.st_stage, i32), (rows.st_c, f64), (rows.st_d, f64))]
        self.warm = eng.zeros((B, self.n), f64)
        self.u = e((B, self.n), f64)
        self.lam = e((B, max(self.m, 1)), f64)
        self.status = e((B,), i32)
        self.iters = e((B,), i32)
        self.resid = e((B, 3), f64)
        self.planned_states = e((B, M, N + 1, nx), f64)
        self.planned_inputs = e((B, N, nu), f64)
        self.next_states = e((B, N + 1, M, nx), f64)
        self.next_inputs = e((B, N, nu), f64)
        self.u_applied = e((B, nu), f64)
        self.u_prev = eng.zeros((B, nu), f64)
        self.has_prev = 0
        self.summary = e((B, nu + 2), f64)
        self.settings_c = settings_c(cfg.solver)
        self.graph = None

    def load(self, x_measured, lin_states, lin_inputs, x_ref, non_blocking: bool = False,
             last_applied=None):
        """Copy the step's inputs (numpy or tensors) into the device buffers:
        x_measured (B, M, nx), lin_states (B, N+1, M, nx), lin_inputs (B, N, nu),
        x_ref (B, M, N+1, nx), and optionally last_applied (B, nu) -- each
        instance's previously applied input, held by the 'hold-previous-input'
        fallback (mpc.py:167-170); without it the fallback applies zeros, as
        the reference does when ``state.last_applied is None``.
        ``non_blocking`` makes copies from pinned host tensors asynchronous on
        the current stream (WavePipeline)."""
        torch = self.eng.torch
        pairs = [(self.x0, x_measured), (self.X, lin_states), (self.U, lin_inputs),
                 (self.xref, x_ref)]
        self.has_prev = 0 if last_applied is None else 1
        if last_applied is not None:
            pairs.append((self.u_prev, last_applied))
        for dst, src in pairs:
            if isinstance(src, np.ndarray):
                dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)))
            else:
                dst.copy_(src, non_blocking=non_blocking)
        self.X[:, 0].copy_(self.x0)  # measurement at stage 0 (mpc.py:120-122)

    def enqueue(self, events=None):
        """All stages for all B instances on the current stream, no host sync.
        ``events`` (5 torch.cuda.Event, optional) are recorded on the stream
        around K-LIN | K-COND (+ rows, soft) | K-QP | K-RS for stage timing."""
        eng, B, N, nx, nu = self.eng, self.B, self.N, self.nx, self.nu
        ctx, sp = eng.ctx, eng.stream_ptr()
        E = eng.E
        M = eng.M

        def mark(i):
            if events is not None:
                events[i].record()

        mark(0)
        # K-LIN over B*N points: linearise along the first N states of each instance
        Xlin = self.X[:, :N]  # (B, N, M, nx) view, contiguous per instance block
        if not Xlin.is_contiguous():
            Xlin = Xlin.contiguous()
        ctx.call("gm_linearize", B * N, Xlin.data_ptr(), self.U.data_ptr(), self.a_self.data_ptr(),
                 self.a_nbr.data_ptr() if E else None, self.b.data_ptr(), self.c.data_ptr(), None,
                 sp)
        mark(1)
        # K-COND: Gamma recursion + H/g reduction in one persistent kernel
        ctx.call("gm_condense_fused", B, N, self.a_self.data_ptr(),
                 self.a_nbr.data_ptr() if E else None, self.b.data_ptr(), self.c.data_ptr(),
                 self.x0.data_ptr(), self.W.data_ptr(), self.ld, self.q.data_ptr(), 0,
                 self.xref.data_ptr(), M * (N + 1) * nx, self.r.data_ptr(), 0,
                 self.uref.data_ptr(), 0, self.H0.data_ptr(), self.g0.data_ptr(), sp)
        rows = self.rows
        if rows.m0:
            p = [t.data_ptr() if t is not None else None for t in self.dev_rows]
            ctx.call("gm_constraint_rows", B, N, self.W.data_ptr(), self.ld, rows.n_in, p[0], p[1],
                     p[2], rows.n_st, p[3], p[4], p[5], p[6], self.C0.data_ptr(),
                     self.d0.data_ptr(), sp)
        if self.ns:
            ctx.call("gm_expand_soft", B, self.n0, self.m0, self.H0.data_ptr(), self.g0.data_ptr(),
                     self.C0.data_ptr(), self.d0.data_ptr(), self.ns, self.idx.data_ptr(),
                     self.rho1.data_ptr(), self.rho2.data_ptr(), self.H.data_ptr(),
                     self.g.data_ptr(), self.C.data_ptr(), self.d.data_ptr(), sp)
        mark(2)
        warm = None
        if self.cfg.warm_start:
            self.warm[:, : N * nu].copy_(self.U.reshape(B, N * nu))
            warm = self.warm.data_ptr()
        ctx.call("gm_solve_qp", B, self.n, self.m, self.H.data_ptr(), self.g.data_ptr(),
                 self.C.data_ptr() if self.m else None, self.d.data_ptr() if self.m else None,
                 warm, ctypes.byref(self.settings_c), self.u.data_ptr(), self.lam.data_ptr(),
                 self.status.data_ptr(), self.iters.data_ptr(), self.resid.data_ptr(), sp)
        mark(3)
        tail = (self.status.data_ptr(), self.iters.data_ptr(), self.X.data_ptr(),
                self.U.data_ptr(), self.X.data_ptr(), self.U.data_ptr(),
                float(self.cfg.sqp_damping),
                0 if self.cfg.fallback == "hold-previous-input" else 1, self.u_prev.data_ptr(),
                self.has_prev, None, self.planned_states.data_ptr(), self.planned_inputs.data_ptr(),
                self.next_states.data_ptr(), self.next_inputs.data_ptr(),
                self.u_applied.data_ptr(), self.summary.data_ptr(), sp)
        if _dev.use_rollout(B * M * (N + 1), nx, nu):  # K-RS by linear rollout (large waves)
            ctx.call("gm_mpc_finish_rollout", B, N, self.a_self.data_ptr(),
                     self.a_nbr.data_ptr() if E else None, self.b.data_ptr(), self.c.data_ptr(),
                     self.x0.data_ptr(), self.u.data_ptr(), self.n, *tail)
        else:
            ctx.call("gm_mpc_finish", B, N, self.W.data_ptr(), self.ld, self.u.data_ptr(), self.n,
                     *tail)
        mark(4)

    def step(self, x_measured, lin_states, lin_inputs, x_ref, last_applied=None) -> BatchResult:
        self.load(x_measured, lin_states, lin_inputs, x_ref, last_applied=last_applied)
        self.enqueue()
        summ = self.summary.cpu().numpy()
        nu = self.nu
        return BatchResult(u_applied=summ[:, :nu].copy(),
                           status=[STATUS_BY_CODE[int(s)] for s in summ[:, nu]],
                           iterations=summ[:, nu + 1].astype(int),
                           next_states=self.next_states, next_inputs=self.next_inputs)


class WavePipeline:
    """A batch run as back-to-back waves of :class:`BatchedMpc`, each wave's
    host->device input copy overlapped with the previous wave's kernels.

    Two BatchedMpc buffer sets per wave size alternate: wave w's inputs are
    copied on a side stream into the set wave w-1 is not using (after that
    set's previous wave has finished), the compute stream waits for the copy,
    runs the wave and queues the D2H of its summary into a per-wave pinned
    buffer; one host synchronisation per :meth:`step`.  Results equal
    ``[BatchedMpc.step(*inp) for inp in inputs]`` wave by wave (same kernels
    on the same data); ``next_states`` / ``next_inputs`` are device copies
    owned by the result."""

    def __init__(self, model, topo, spec, cfg: MpcConfig, sizes, device=None):
        self.sizes = [int(n) for n in sizes]
        self.sets = {n: [BatchedMpc(model, topo, spec, cfg, n, device) for _ in range(2)]
                     for n in sorted(set(self.sizes))}
        first = next(iter(self.sets.values()))[0]
        self.torch = torch = first.eng.torch
        self.device = first.eng.device
        self.nu = first.nu
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.summ = [torch.empty((n, self.nu + 2), dtype=torch.float64).pin_memory() for n in self.sizes]
        self.done = {}

    def step(self, inputs) -> list:
        """inputs: one (x_measured, lin_states, lin_inputs, x_ref) tuple of
        pinned host tensors per wave, shaped for that wave's size."""
        torch = self.torch
        if len(inputs) != len(self.sizes):
            raise ValueError(f"expected {len(self.sizes)} waves of inputs, got {len(inputs)}")
        cs = torch.cuda.current_stream(self.device)
        turn = {n: 0 for n in self.sets}
        nexts = []
        for w, (n, inp) in enumerate(zip(self.sizes, inputs)):
            bm = self.sets[n][turn[n] & 1]
            turn[n] += 1
            with torch.cuda.stream(self.copy_stream):
                prev = self.done.get(id(bm))
                if prev is not None:
                    self.copy_stream.wait_event(prev)  # the set's previous wave is finished
                bm.load(*inp, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(self.copy_stream)
            cs.wait_event(loaded)
            bm.enqueue()
            self.summ[w].copy_(bm.summary, non_blocking=True)
            nexts.append((bm.next_states.clone(), bm.next_inputs.clone()))
            done = torch.cuda.Event()
            done.record(cs)
            self.done[id(bm)] = done
        cs.synchronize()
        out = []
        for w, (ns, ni) in enumerate(nexts):
            summ = self.summ[w].numpy()
            nu = self.nu
            out.append(BatchResult(u_applied=summ[:, :nu].copy(),
                                   status=[STATUS_BY_CODE[int(s)] for s in summ[:, nu]],
                                   iterations=summ[:, nu + 1].astype(int),
                                   next_states=ns, next_inputs=ni))
        return out
