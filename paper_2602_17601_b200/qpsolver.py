"""Dense interior-point QP solver -- reference-compatible API on the GPU.

Mirrors ``gnnmpc/qpsolver.py``: ``QpStatus`` / ``QpProblem`` /
``SolverSettings`` / ``QpSolution`` / ``solve_qp`` (``:24-235``).  The solve
runs in the fp64 one-CTA-per-QP kernel K-QP (``csrc/k_qp.cu``);
``solve_qp_batched`` exposes the batched form (independent QPs, one CTA each).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import device as _dev
from ._runtime import QP_STATUS_NAMES, QpSettingsC
from .graph import chain_topology


class QpStatus(Enum):
    OPTIMAL = "optimal"
    MAX_ITERATIONS = "max_iterations"
    PRIMAL_INFEASIBLE = "primal_infeasible"
    NUMERICAL_FAILURE = "numerical_failure"


STATUS_BY_CODE = tuple(QpStatus(v) for v in QP_STATUS_NAMES)


@dataclass
class QpProblem:
    """``min u'Hu + g'u  s.t.  C u <= d`` (validation ``qpsolver.py:38-52``)."""

    h: np.ndarray
    g: np.ndarray
    c: np.ndarray
    d: np.ndarray

    def __post_init__(self):
        self.h = np.asarray(self.h, dtype=float)
        self.g = np.asarray(self.g, dtype=float).reshape(-1)
        n = self.g.shape[0]
        if self.h.shape != (n, n):
            raise ValueError("H must be square and match g")
        if float(np.max(np.abs(self.h - self.h.T))) > 1e-12 * max(1.0, float(np.max(np.abs(self.h)))):
            raise ValueError("H must be symmetric")
        if self.c is None:
            self.c = np.zeros((0, n))
            self.d = np.zeros(0)
        self.c = np.atleast_2d(np.asarray(self.c, dtype=float)) if np.size(self.c) else np.zeros((0, n))
        self.d = np.asarray(self.d, dtype=float).reshape(-1)
        if self.c.shape != (self.d.shape[0], n):
            raise ValueError("C/d shape mismatch")

    @property
    def n(self) -> int:
        return self.g.shape[0]

    @property
    def m(self) -> int:
        return self.d.shape[0]

    def objective(self, u: np.ndarray) -> float:
        return float(u @ self.h @ u + self.g @ u)


@dataclass
class SolverSettings:
    tolerance: float = 1e-8
    max_iterations: int = 50
    regularization: float = 1e-9
    fraction_to_boundary: float = 0.995
    warm_start: np.ndarray | None = None

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")

    def as_c(self) -> QpSettingsC:
        return settings_c(self)


def settings_c(s) -> QpSettingsC:
    """The C struct of any SolverSettings-like object (ours or the
    reference's, qpsolver.py:66-76)."""
    return QpSettingsC(float(s.tolerance), int(s.max_iterations), float(s.regularization),
                       float(s.fraction_to_boundary))


@dataclass
class QpSolution:
    u: np.ndarray
    duals: np.ndarray
    status: QpStatus
    iterations: int
    stationarity: float
    primal_infeas: float
    complementarity: float


_topo1 = chain_topology(1)


def solve_qp_device(eng, H, g, C, d, warm, settings: SolverSettings, B: int = 1):
    """K-QP on device tensors (H (B,n,n), g (B,n), C (B,m,n), d (B,m)).
    Returns device tensors (u, lam, status, iterations, resid)."""
    n = int(g.shape[-1])
    m = int(d.shape[-1])
    u = eng.empty((B, n), np.float64)
    lam = eng.empty((B, max(m, 1)), np.float64)
    st = eng.empty((B,), np.int32)
    it = eng.empty((B,), np.int32)
    rs = eng.empty((B, 3), np.float64)
    cs = settings_c(settings)
    eng.ctx.call("gm_solve_qp", B, n, m, H.data_ptr(), g.data_ptr(),
                 C.data_ptr() if C.numel() else None, d.data_ptr() if d.numel() else None,
                 warm.data_ptr() if warm is not None else None, ctypes.byref(cs), u.data_ptr(),
                 lam.data_ptr(), st.data_ptr(), it.data_ptr(), rs.data_ptr(), eng.stream_ptr())
    return u, lam[:, :m], st, it, rs


def solve_qp(problem: QpProblem, settings: SolverSettings | None = None) -> QpSolution:
    """Predictor-corrector interior point (``qpsolver.py:112-235``) on the GPU;
    deterministic, returns the best iterate when the iteration cap is hit."""
    s = settings or SolverSettings()
    p = problem
    n = p.n
    warm = None
    if s.warm_start is not None:
        warm = np.asarray(s.warm_start, dtype=float)
        if warm.shape != (n,):
            raise ValueError("warm start dimension mismatch")
    eng = _dev.engine(_topo1)
    H = eng.h2d(p.h, np.float64)
    g = eng.h2d(p.g, np.float64)
    C = eng.h2d(p.c.reshape(p.m, n), np.float64)
    d = eng.h2d(p.d, np.float64)
    w = eng.h2d(warm, np.float64) if warm is not None else None
    u, lam, st, it, rs = solve_qp_device(eng, H, g, C, d, w, s)
    rs = rs.cpu().numpy()[0]
    return QpSolution(u=u.cpu().numpy()[0], duals=lam.cpu().numpy()[0],
                      status=STATUS_BY_CODE[int(st.cpu().numpy()[0])],
                      iterations=int(it.cpu().numpy()[0]), stationarity=float(rs[0]),
                      primal_infeas=float(rs[1]), complementarity=float(rs[2]))


def solve_qp_batched(H, g, C, d, settings: SolverSettings | None = None, warm=None):
    """Independent QPs with shared shapes, one CTA each.  Arrays are stacked on
    a leading batch axis; returns a list of ``QpSolution``."""
    s = settings or SolverSettings()
    H = np.asarray(H, dtype=float)
    B, n, _ = H.shape
    g = np.asarray(g, dtype=float).reshape(B, n)
    d = np.asarray(d, dtype=float).reshape(B, -1)
    m = d.shape[1]
    C = np.asarray(C, dtype=float).reshape(B, m, n)
    eng = _dev.engine(_topo1)
    w = eng.h2d(np.asarray(warm, dtype=float).reshape(B, n), np.float64) if warm is not None else None
    u, lam, st, it, rs = solve_qp_device(eng, eng.h2d(H, np.float64), eng.h2d(g, np.float64),
                                         eng.h2d(C, np.float64), eng.h2d(d, np.float64), w, s, B)
    u, lam, st, it, rs = (t.cpu().numpy() for t in (u, lam, st, it, rs))
    return [QpSolution(u[b], lam[b], STATUS_BY_CODE[int(st[b])], int(it[b]), float(rs[b, 0]),
                       float(rs[b, 1]), float(rs[b, 2])) for b in range(B)]
