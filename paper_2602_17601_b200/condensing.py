"""Structure-exploiting condensing -- reference-compatible API on the GPU.

Mirrors ``gnnmpc/condensing.py``: ``StateConstraint`` / ``OcpSpec``
(``:45-129``), ``stage_input_box`` (``:132-138``),
``cost_to_standard_form`` (``:141-155``), ``condense_gammas``
(``:182-228``), ``CondensedQp`` / ``condense_ocp`` (``:298-406``),
``reconstruct_states`` (``:409-416``), ``expand_soft_constraints``
(``:419-439``).  Conventions kept: the QP objective is ``u'Hu + g'u`` (no 1/2,
so g carries the factor-2 term), constraint rows are input rows first
(stage-major), then state rows by node ascending and stage ascending.

The recursion (K-REC), the H/g contraction (K-HG), the constraint mapping and
the soft expansion run in ``csrc/k_condense.cu``.  Gamma lives on the device
as one fp32 work array (Gamma_u columns + a Gamma_x column); the arrays
returned to callers are read-only fp64 NumPy views, and passing them back
(``condense_ocp(..., gammas=...)``, ``reconstruct_states``) reuses the device
copy instead of re-uploading.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np

from . import device as _dev
from .errors import ConfigurationError
from .graph import GraphTopology, chain_topology

__all__ = [
    "ConfigurationError", "StateConstraint", "OcpSpec", "stage_input_box", "StandardFormCost",
    "cost_to_standard_form", "CondensedQp", "condense_gammas", "condense_ocp",
    "reconstruct_states", "expand_soft_constraints", "min_eig_sym", "local_hessian_gradient",
    "LocalCondensed", "condense_local", "assemble_qp",
]


def min_eig_sym(A: np.ndarray) -> float:
    return float(np.linalg.eigvalsh(0.5 * (A + A.T))[0])


@dataclass
class StateConstraint:
    """Half-space rows ``C x_i[k] <= d`` on one node at one stage (``:45-63``)."""

    node: int
    stage: int
    c: np.ndarray
    d: np.ndarray
    soft: bool = False
    rho1: float = 1e3
    rho2: float = 1e4

    def __post_init__(self):
        self.c = np.atleast_2d(np.asarray(self.c, dtype=float))
        self.d = np.atleast_1d(np.asarray(self.d, dtype=float))
        if self.c.shape[0] != self.d.shape[0]:
            raise ConfigurationError("constraint row count does not match bound length")
        if self.soft and self.rho2 <= 0:
            raise ConfigurationError("soft constraints need rho2 > 0")


@dataclass
class OcpSpec:
    """Tracking OCP data (``condensing.py:66-129``).

    ``freeze()`` marks the cost / reference arrays read-only; frozen arrays are
    uploaded to the GPU once and reused across ``mpc_step`` calls (unfrozen
    arrays are re-uploaded on every call, which honours in-place edits)."""

    topology: GraphTopology
    horizon: int
    q: np.ndarray
    x_ref: np.ndarray
    r: np.ndarray
    u_ref: np.ndarray
    input_constraints: list | None = None
    state_constraints: list = field(default_factory=list)

    def __post_init__(self):
        M = self.topology.node_count
        N = self.horizon
        self.q = np.asarray(self.q, dtype=float)
        self.x_ref = np.asarray(self.x_ref, dtype=float)
        self.r = np.asarray(self.r, dtype=float)
        self.u_ref = np.asarray(self.u_ref, dtype=float)
        nx = self.q.shape[-1]
        if self.q.shape != (M, N + 1, nx, nx):
            raise ConfigurationError("q must be (M, N+1, n_state, n_state)")
        if self.x_ref.shape != (M, N + 1, nx):
            raise ConfigurationError("x_ref must be (M, N+1, n_state)")
        nu = self.r.shape[-1]
        if self.r.shape != (N, nu, nu):
            raise ConfigurationError("r must be (N, n_u, n_u)")
        if self.u_ref.shape != (N, nu):
            raise ConfigurationError("u_ref must be (N, n_u)")
        if self.input_constraints is not None:
            if len(self.input_constraints) != N:
                raise ConfigurationError("need one input constraint pair per stage")
            norm = []
            for C, d in self.input_constraints:
                C = np.atleast_2d(np.asarray(C, dtype=float))
                d = np.atleast_1d(np.asarray(d, dtype=float))
                if C.shape != (d.shape[0], nu):
                    raise ConfigurationError("input constraint shape mismatch")
                norm.append((C, d))
            self.input_constraints = norm
        for sc in self.state_constraints:
            if not 0 <= sc.node < M or not 0 <= sc.stage <= N:
                raise ConfigurationError("state constraint node/stage out of range")
            if sc.c.shape[1] != nx:
                raise ConfigurationError("state constraint column count != n_state")

    @property
    def n_state(self) -> int:
        return self.q.shape[-1]

    @property
    def n_u(self) -> int:
        return self.r.shape[-1]

    def validate_costs(self) -> None:
        qs = 0.5 * (self.q + np.swapaxes(self.q, -1, -2))
        if float(np.min(np.linalg.eigvalsh(qs))) < -1e-10:
            raise ConfigurationError("state cost has eigenvalue below -1e-10")
        rs = 0.5 * (self.r + np.swapaxes(self.r, -1, -2))
        if float(np.min(np.linalg.eigvalsh(rs))) < 1e-12:
            raise ConfigurationError("input cost is not positive definite")

    def freeze(self) -> "OcpSpec":
        """Make the spec immutable (arrays read-only, constraint lists tuples) so
        its device copy can be cached across steps."""
        for a in (self.q, self.x_ref, self.r, self.u_ref):
            a.flags.writeable = False
        if self.input_constraints is not None:
            for C, d in self.input_constraints:
                C.flags.writeable = False
                d.flags.writeable = False
            self.input_constraints = tuple(self.input_constraints)
        for sc in self.state_constraints:
            sc.c.flags.writeable = False
            sc.d.flags.writeable = False
        self.state_constraints = tuple(self.state_constraints)
        object.__setattr__(self, "_frozen", True)
        return self


def stage_input_box(n_u: int, lo, hi):
    """Box ``lo <= u <= hi`` as half-space rows ``[I; -I] u <= [hi; -lo]``."""
    lo = np.broadcast_to(np.asarray(lo, dtype=float), (n_u,))
    hi = np.broadcast_to(np.asarray(hi, dtype=float), (n_u,))
    return np.vstack([np.eye(n_u), -np.eye(n_u)]), np.concatenate([hi, -lo])


@dataclass
class StandardFormCost:
    q_blocks: np.ndarray
    q_lin: np.ndarray
    r_blocks: np.ndarray
    r_lin: np.ndarray


def cost_to_standard_form(spec) -> StandardFormCost:
    """q = -2 Q x_ref, r = -2 R u_ref (``:152-155``).  Host-side data prep for
    callers; the device path forms the same terms inside K-HG."""
    q_lin = -2.0 * np.einsum("mkab,mkb->mka", spec.q, spec.x_ref)
    r_lin = -2.0 * np.einsum("kab,kb->ka", spec.r, spec.u_ref)
    return StandardFormCost(spec.q, q_lin, spec.r, r_lin)


@dataclass
class CondensedQp:
    h: np.ndarray
    g: np.ndarray
    c: np.ndarray
    d: np.ndarray
    soft: np.ndarray
    rho1: np.ndarray
    rho2: np.ndarray


# ---------------------------------------------------------------------------
# spec -> device
# ---------------------------------------------------------------------------

@dataclass
class SpecRows:
    """Constraint rows flattened in the reference's stacking order."""

    n_in: int
    in_stage: np.ndarray
    in_c: np.ndarray
    in_d: np.ndarray
    n_st: int
    st_node: np.ndarray
    st_stage: np.ndarray
    st_c: np.ndarray
    st_d: np.ndarray
    soft: np.ndarray
    rho1: np.ndarray
    rho2: np.ndarray

    @property
    def m0(self) -> int:
        return self.n_in + self.n_st

    @property
    def soft_idx(self) -> np.ndarray:
        return np.flatnonzero(self.soft).astype(np.int32)


def spec_rows(spec, nx: int, nu: int) -> SpecRows:
    """Input rows stage-major (``:312-323``), then state rows grouped by node
    ascending, stage ascending within a node (stable, ``:265-267``)."""
    in_stage, in_c, in_d = [], [], []
    if spec.input_constraints is not None:
        for k, (Ck, dk) in enumerate(spec.input_constraints):
            Ck = np.atleast_2d(np.asarray(Ck, dtype=float))
            in_stage.extend([k] * Ck.shape[0])
            in_c.append(Ck)
            in_d.append(np.atleast_1d(np.asarray(dk, dtype=float)))
    n_in = len(in_stage)
    scs = sorted(spec.state_constraints, key=lambda s: (s.node, s.stage))
    st_node, st_stage, st_c, st_d, soft, r1, r2 = [], [], [], [], [], [], []
    for sc in scs:
        cc = np.atleast_2d(np.asarray(sc.c, dtype=float))
        rows = cc.shape[0]
        st_node.extend([sc.node] * rows)
        st_stage.extend([sc.stage] * rows)
        st_c.append(cc)
        st_d.append(np.atleast_1d(np.asarray(sc.d, dtype=float)))
        soft.extend([bool(sc.soft)] * rows)
        r1.extend([float(sc.rho1)] * rows)
        r2.extend([float(sc.rho2)] * rows)
    n_st = len(st_node)
    return SpecRows(
        n_in=n_in, in_stage=np.asarray(in_stage, dtype=np.int32),
        in_c=np.vstack(in_c) if in_c else np.zeros((0, nu)),
        in_d=np.concatenate(in_d) if in_d else np.zeros(0),
        n_st=n_st, st_node=np.asarray(st_node, dtype=np.int32),
        st_stage=np.asarray(st_stage, dtype=np.int32),
        st_c=np.vstack(st_c) if st_c else np.zeros((0, nx)),
        st_d=np.concatenate(st_d) if st_d else np.zeros(0),
        soft=np.concatenate([np.zeros(n_in, dtype=bool), np.asarray(soft, dtype=bool)]),
        rho1=np.concatenate([np.zeros(n_in), np.asarray(r1, dtype=float)]),
        rho2=np.concatenate([np.zeros(n_in), np.asarray(r2, dtype=float)]))


class DeviceSpec:
    """Everything of an OcpSpec the device path reads, uploaded once."""

    def __init__(self, eng, spec, nx: int, nu: int, local_nodes=None, node_map=None):
        """``local_nodes`` (global ids, ascending) / ``node_map`` (global id ->
        local id, -1 elsewhere) restrict the per-node arrays to one rank's
        local nodes of a node partition (partition.py); the constraint rows
        keep the global order (sorted by global node id) with each state
        row's node mapped to its local id (rows of non-local nodes point at
        local node 0 and are masked by the caller)."""
        f64, i32 = np.float64, np.int32
        self.rows = rows = spec_rows(spec, nx, nu)
        q, x_ref = spec.q, spec.x_ref
        if local_nodes is not None:
            q, x_ref = np.asarray(q)[local_nodes], np.asarray(x_ref)[local_nodes]
            if rows.n_st:
                loc = np.asarray(node_map)[rows.st_node]
                rows.st_node = np.where(loc >= 0, loc, 0).astype(np.int32)
        self.q = eng.h2d(q, f64)
        self.x_ref = eng.h2d(x_ref, f64)
        self.r = eng.h2d(spec.r, f64)
        self.u_ref = eng.h2d(spec.u_ref, f64)
        self.in_stage = eng.h2d(rows.in_stage, i32) if rows.n_in else None
        self.in_c = eng.h2d(rows.in_c, f64) if rows.n_in else None
        self.in_d = eng.h2d(rows.in_d, f64) if rows.n_in else None
        self.st_node = eng.h2d(rows.st_node, i32) if rows.n_st else None
        self.st_stage = eng.h2d(rows.st_stage, i32) if rows.n_st else None
        self.st_c = eng.h2d(rows.st_c, f64) if rows.n_st else None
        self.st_d = eng.h2d(rows.st_d, f64) if rows.n_st else None
        self.soft_idx = rows.soft_idx
        self.ns = int(self.soft_idx.size)
        if self.ns:
            self.idx = eng.h2d(self.soft_idx, i32)
            self.rho1 = eng.h2d(rows.rho1[self.soft_idx], f64)
            self.rho2 = eng.h2d(rows.rho2[self.soft_idx], f64)


def device_spec(eng, spec, nx: int, nu: int) -> DeviceSpec:
    """Device copy of ``spec``; cached per engine for frozen specs
    (``OcpSpec.freeze``), rebuilt on every call otherwise.  Specs produced by a
    tracking provider (``tracking.tracking_spec_provider``) share frozen cost /
    constraint arrays and carry the provider's static token: their upload is
    cached under the token and only x_ref is copied in on each call."""
    token = getattr(spec, "_static_token", None)
    if token is not None:
        key = ("spec-token", id(token), nx, nu)
        hit = eng.cache.get(key)
        if hit is not None and hit[0]() is token:
            ds = hit[1]
            src = eng.torch.from_numpy(np.ascontiguousarray(spec.x_ref, dtype=np.float64))
            ds.x_ref.copy_(src.reshape(ds.x_ref.shape))
            return ds
        ds = DeviceSpec(eng, spec, nx, nu)
        eng.cache[key] = (weakref.ref(token), ds)
        weakref.finalize(token, eng.cache.pop, key, None)
        return ds
    if not getattr(spec, "_frozen", False):
        return DeviceSpec(eng, spec, nx, nu)
    key = ("spec", id(spec), nx, nu)
    hit = eng.cache.get(key)
    if hit is not None and hit[0]() is spec:
        return hit[1]
    ds = DeviceSpec(eng, spec, nx, nu)
    eng.cache[key] = (weakref.ref(spec), ds)
    weakref.finalize(spec, eng.cache.pop, key, None)
    return ds


def _ptr(t):
    return None if t is None or t.numel() == 0 else t.data_ptr()


def cost_device(eng, ds: DeviceSpec, W, ld, N, H0, g0, partial=0):
    """K-HG: H0 (n0,n0), g0 (n0) fp64 from the device work array W."""
    eng.ctx.call("gm_condense_cost", 1, N, W.data_ptr(), ld, ds.q.data_ptr(), 0,
                 ds.x_ref.data_ptr(), 0, ds.r.data_ptr(), 0, ds.u_ref.data_ptr(), 0,
                 H0.data_ptr(), g0.data_ptr(), int(partial), eng.stream_ptr())


def fused_device(eng, ds: DeviceSpec, a_self, a_nbr, b, c, x0, W, ld, N, H0, g0):
    """K-COND: Gamma recursion into W and H0, g0 in one persistent kernel."""
    eng.ctx.call("gm_condense_fused", 1, N, a_self.data_ptr(), _ptr(a_nbr), b.data_ptr(),
                 c.data_ptr(), x0.data_ptr(), W.data_ptr(), ld, ds.q.data_ptr(), 0,
                 ds.x_ref.data_ptr(), 0, ds.r.data_ptr(), 0, ds.u_ref.data_ptr(), 0,
                 H0.data_ptr(), g0.data_ptr(), eng.stream_ptr())


def rows_device(eng, ds: DeviceSpec, W, ld, N, C0, d0):
    """K-CON: constraint rows C0 (m0, n0), d0 (m0) fp64."""
    rows = ds.rows
    if rows.m0 == 0:
        return
    eng.ctx.call("gm_constraint_rows", 1, N, W.data_ptr(), ld, rows.n_in, _ptr(ds.in_stage),
                 _ptr(ds.in_c), _ptr(ds.in_d), rows.n_st, _ptr(ds.st_node), _ptr(ds.st_stage),
                 _ptr(ds.st_c), _ptr(ds.st_d), C0.data_ptr(), d0.data_ptr(), eng.stream_ptr())


# ---------------------------------------------------------------------------
# Gamma work array registry (device copy reuse for returned views)
# ---------------------------------------------------------------------------

_gamma_registry: dict = {}


def _register_gammas(gu, gx, W, ld, N, nu):
    key = id(gu)
    _gamma_registry[key] = (weakref.ref(gu), weakref.ref(gx), W, ld, N, nu)
    weakref.finalize(gu, _gamma_registry.pop, key, None)


def _lookup_gammas(gammas, eng):
    gu, gx = gammas
    hit = _gamma_registry.get(id(gu))
    if hit is None:
        return None
    rgu, rgx, W, ld, N, nu = hit
    if rgu() is gu and rgx() is gx and W.device == eng.device:
        return W, ld
    return None


def _upload_gammas(eng, gu, gx, N, nx, nu):
    """Pack host (gamma_u, gamma_x) into the device work-array layout."""
    from ._runtime import lib

    M = gu.shape[0]
    ld = lib().gm_gamma_ld(N, nu)
    Wh = np.zeros((M, N + 1, nx, ld), dtype=np.float32)
    Wh[..., : N * nu] = gu
    Wh[..., N * nu] = gx
    return eng.h2d(Wh, np.float32), ld


def lin_blocks(lin, eng):
    """Device blocks of any LinearizedDynamics-like object (ours or the
    reference's NumPy dataclass)."""
    if hasattr(lin, "device_blocks"):
        return lin.device_blocks(eng)
    return tuple(eng.h2d(np.asarray(getattr(lin, k)), np.float64 if k == "c" else np.float32)
                 for k in ("a_self", "a_nbr", "b", "c"))


def gammas_device(eng, lin, x0, N, nx, nu):
    """Run K-REC; returns (W, ld) with W (M, N+1, nx, ld) fp32 on the device."""
    from ._runtime import lib

    ld = lib().gm_gamma_ld(N, nu)
    a_self, a_nbr, b, c = lin
    W = eng.empty((eng.M, N + 1, nx, ld), np.float32)
    eng.ctx.call("gm_condense_gammas", 1, N, a_self.data_ptr(), _ptr(a_nbr), b.data_ptr(),
                 c.data_ptr(), x0.data_ptr(), W.data_ptr(), ld, eng.stream_ptr())
    return W, ld


def _materialise(W, N, nu):
    Wn = W.double().cpu().numpy()
    Wn.flags.writeable = False
    return Wn[..., : N * nu], Wn[..., N * nu]


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------

def condense_gammas(lin, x0, threads: int = 1):
    """Per-node prediction maps (``condensing.py:182-228``) computed by K-REC.

    Returns ``(gamma_u (M, N+1, nx, N*nu), gamma_x (M, N+1, nx))``.  ``threads``
    is accepted for API compatibility; the GPU parallelises over nodes and
    columns regardless (results are bitwise independent of it, like the
    reference's)."""
    topo = lin.topology
    N, nx, nu = lin.horizon, lin.n_state, lin.n_u
    eng = _dev.engine(topo)
    eng.set_dims(nx, nu)
    blocks = lin_blocks(lin, eng)
    x0d = eng.h2d(np.asarray(x0, dtype=float).reshape(topo.node_count, nx), np.float64)
    W, ld = gammas_device(eng, blocks, x0d, N, nx, nu)
    gu, gx = _materialise(W, N, nu)
    _register_gammas(gu, gx, W, ld, N, nu)
    return gu, gx


def condense_ocp(spec, lin, x0, threads: int = 1, gammas=None) -> CondensedQp:
    """Condensed QP ``min u'Hu + g'u s.t. Cu <= d`` (``condensing.py:363-406``)."""
    from ._runtime import lib

    topo = spec.topology
    N, nx, nu = spec.horizon, spec.n_state, spec.n_u
    eng = _dev.engine(topo)
    eng.set_dims(nx, nu)
    if gammas is not None:
        hit = _lookup_gammas(gammas, eng)
        if hit is None:
            W, ld = _upload_gammas(eng, np.asarray(gammas[0]), np.asarray(gammas[1]), N, nx, nu)
        else:
            W, ld = hit
    n0 = N * nu
    ds = device_spec(eng, spec, nx, nu)
    rows = ds.rows
    H0 = eng.empty((n0, n0), np.float64)
    g0 = eng.empty((n0,), np.float64)
    if gammas is None:  # K-COND: recursion and cost reduction fused
        a_self, a_nbr, b, c = lin_blocks(lin, eng)
        x0d = eng.h2d(np.asarray(x0, dtype=float).reshape(topo.node_count, nx), np.float64)
        ld = lib().gm_gamma_ld(N, nu)
        W = eng.empty((eng.M, N + 1, nx, ld), np.float32)
        fused_device(eng, ds, a_self, a_nbr, b, c, x0d, W, ld, N, H0, g0)
    else:
        cost_device(eng, ds, W, ld, N, H0, g0)
    C0 = eng.empty((rows.m0, n0), np.float64)
    d0 = eng.empty((rows.m0,), np.float64)
    rows_device(eng, ds, W, ld, N, C0, d0)
    return CondensedQp(h=H0.cpu().numpy(), g=g0.cpu().numpy(), c=C0.cpu().numpy(),
                       d=d0.cpu().numpy(), soft=rows.soft.copy(), rho1=rows.rho1.copy(),
                       rho2=rows.rho2.copy())


def expand_soft_device(eng, n0, m0, H0, g0, C0, d0, soft_idx, rho1, rho2):
    """Device soft-constraint expansion; returns (H, g, C, d) tensors."""
    ns = int(soft_idx.size)
    n, m = n0 + ns, m0 + ns
    H = eng.empty((n, n), np.float64)
    g = eng.empty((n,), np.float64)
    C = eng.empty((m, n), np.float64)
    d = eng.empty((m,), np.float64)
    idx = eng.h2d(soft_idx, np.int32)
    r1 = eng.h2d(rho1, np.float64)
    r2 = eng.h2d(rho2, np.float64)
    eng.ctx.call("gm_expand_soft", 1, n0, m0, H0.data_ptr(), g0.data_ptr(), _ptr(C0), _ptr(d0), ns,
                 idx.data_ptr(), r1.data_ptr(), r2.data_ptr(), H.data_ptr(), g.data_ptr(),
                 C.data_ptr(), d.data_ptr(), eng.stream_ptr())
    return H, g, C, d


_qp_topo = chain_topology(1)


def expand_soft_constraints(qp: CondensedQp):
    """One penalised slack per soft row (``condensing.py:419-439``).
    Returns ``(H, g, C, d, n_original)``."""
    idx = np.flatnonzero(qp.soft)
    n = qp.h.shape[0]
    if idx.size == 0:
        return qp.h, qp.g, qp.c, qp.d, n
    eng = _dev.engine(_qp_topo)
    m0 = qp.c.shape[0]
    H, g, C, d = expand_soft_device(
        eng, n, m0, eng.h2d(qp.h, np.float64), eng.h2d(qp.g, np.float64),
        eng.h2d(qp.c, np.float64), eng.h2d(qp.d, np.float64), idx.astype(np.int32),
        np.asarray(qp.rho1, dtype=float)[idx], np.asarray(qp.rho2, dtype=float)[idx])
    return H.cpu().numpy(), g.cpu().numpy(), C.cpu().numpy(), d.cpu().numpy(), n


def reconstruct_states(gamma_u, gamma_x, u) -> np.ndarray:
    """Planned trajectories ``x^i = Gamma_u^i u + Gamma_x^i`` (``:409-416``);
    accepts all-node (M, N+1, nx, N*nu) or single-node (N+1, nx, N*nu) maps."""
    u = np.asarray(u, dtype=float).reshape(-1)
    gu = np.asarray(gamma_u)
    single = gu.ndim == 3
    if single:
        gu = gu[None]
    gx = np.asarray(gamma_x)
    if single:
        gx = gx[None]
    M, Np1, nx, n0 = gu.shape
    N = Np1 - 1
    nu = n0 // N if N else 1
    eng = _dev.engine(_qp_topo)  # one-node graph: every node is an "instance"
    eng.set_dims(nx, nu)
    hit = None if single else _lookup_gammas((gamma_u, gamma_x), eng)
    if hit is None:
        W, ld = _upload_gammas(eng, gu, gx, N, nx, nu)
    else:
        W, ld = hit
    ud = eng.h2d(u, np.float64)
    x = eng.empty((M, N + 1, nx), np.float64)
    eng.ctx.call("gm_reconstruct_states", M, N, W.data_ptr(), ld, ud.data_ptr(), 0, x.data_ptr(),
                 eng.stream_ptr())
    out = x.cpu().numpy()
    return out[0] if single else out


# ---------------------------------------------------------------------------
# per-node condensing (condensing.py:231-360): each node's H^i, g^i and
# constraint rows, and their assembly -- the paper's Eqs. (16)-(17)
# ---------------------------------------------------------------------------

@dataclass
class LocalCondensed:
    """One node's condensed quantities (``condensing.py:246-260``)."""

    node: int
    gamma_u: np.ndarray  # (N+1, n_state, N*n_u)
    gamma_x: np.ndarray  # (N+1, n_state)
    h: np.ndarray  # (N*n_u, N*n_u)
    g: np.ndarray  # (N*n_u,)
    c_rows: np.ndarray  # (rows, N*n_u)
    d_rows: np.ndarray  # (rows,)
    soft: np.ndarray  # (rows,) bool
    rho1: np.ndarray  # (rows,)
    rho2: np.ndarray  # (rows,)
    # device copies of every node's (h, g) of the condense_local call that
    # produced this node, and its index there (assemble_qp sums on the device
    # without re-uploading)
    _dev: tuple | None = field(default=None, repr=False, compare=False)


def node_hessians_device(eng, W, ld, N, q, q_lin):
    """K-NHG: per-node (H^i, g^i) of every node of the engine's graph on the
    device: H (M, n0, n0), g (M, n0) fp64 tensors."""
    nu = eng._dims[1] if eng._dims else None
    n0 = N * nu
    H = eng.empty((eng.M, n0, n0), np.float64)
    g = eng.empty((eng.M, n0), np.float64)
    eng.ctx.call("gm_node_hessians", 1, N, W.data_ptr(), ld, q.data_ptr(), 0, q_lin.data_ptr(), 0,
                 H.data_ptr(), g.data_ptr(), eng.stream_ptr())
    return H, g


def local_hessian_gradient(gamma_u, gamma_x, q_blocks, q_lin):
    """One node's Hessian and gradient contribution (``condensing.py:231-243``):
    ``0.5 (h + h')`` with ``h = sum_k Gu_k' Q_k Gu_k`` and
    ``g = sum_k Gu_k' (2 Q_k Gx_k + q_lin_k)``, on the GPU (K-NHG).
    gamma_u (N+1, n_state, N*n_u), gamma_x (N+1, n_state), q_blocks
    (N+1, n_state, n_state), q_lin (N+1, n_state)."""
    gu = np.asarray(gamma_u, dtype=float)
    gx = np.asarray(gamma_x, dtype=float)
    S1, nx, n0 = gu.shape
    N = S1 - 1
    if N < 1 or n0 % N:
        raise ConfigurationError("gamma_u must be (N+1, n_state, N*n_u) with N >= 1")
    nu = n0 // N
    if gx.shape != (S1, nx):
        raise ConfigurationError("gamma_x must be (N+1, n_state)")
    eng = _dev.engine(_qp_topo)
    eng.set_dims(nx, nu)
    W, ld = _upload_gammas(eng, gu[None], gx[None], N, nx, nu)
    q = eng.h2d(np.asarray(q_blocks, dtype=float).reshape(1, S1, nx, nx), np.float64)
    ql = eng.h2d(np.asarray(q_lin, dtype=float).reshape(1, S1, nx), np.float64)
    H, g = node_hessians_device(eng, W, ld, N, q, ql)
    return H[0].cpu().numpy(), g[0].cpu().numpy()


def condense_local(spec, lin, x0) -> list:
    """Per-node condensing (``condensing.py:285-295``): the Gamma recursion
    (K-REC), every node's cost contribution (K-NHG) and its state-constraint
    rows mapped to input space (K-CON), all on the GPU."""
    topo = spec.topology
    N, nx, nu = spec.horizon, spec.n_state, spec.n_u
    M, n0 = topo.node_count, N * nu
    eng = _dev.engine(topo)
    eng.set_dims(nx, nu)
    blocks = lin_blocks(lin, eng)
    x0d = eng.h2d(np.asarray(x0, dtype=float).reshape(M, nx), np.float64)
    W, ld = gammas_device(eng, blocks, x0d, N, nx, nu)
    cost = cost_to_standard_form(spec)
    q = eng.h2d(spec.q, np.float64)
    ql = eng.h2d(cost.q_lin, np.float64)
    Hd, gd = node_hessians_device(eng, W, ld, N, q, ql)
    rows = spec_rows(spec, nx, nu)
    C = d = None
    if rows.n_st:
        f64, i32 = np.float64, np.int32
        Cd = eng.empty((rows.n_st, n0), f64)
        dd = eng.empty((rows.n_st,), f64)
        # keep the uploads referenced until the kernel is enqueued (a bare
        # .data_ptr() of a temporary lets the allocator hand its block to the
        # next upload)
        sn, ss = eng.h2d(rows.st_node, i32), eng.h2d(rows.st_stage, i32)
        sc, sd = eng.h2d(rows.st_c, f64), eng.h2d(rows.st_d, f64)
        eng.ctx.call("gm_constraint_rows", 1, N, W.data_ptr(), ld, 0, None, None, None, rows.n_st,
                     sn.data_ptr(), ss.data_ptr(), sc.data_ptr(), sd.data_ptr(),
                     Cd.data_ptr(), dd.data_ptr(), eng.stream_ptr())
        C, d = Cd.cpu().numpy(), dd.cpu().numpy()
    gu, gx = _materialise(W, N, nu)
    H, g = Hd.cpu().numpy(), gd.cpu().numpy()
    # state rows are grouped by node ascending, stage ascending (spec_rows),
    # exactly the per-node order of _node_constraint_rows (:263-282)
    st_node = rows.st_node
    bounds = np.searchsorted(st_node, np.arange(M + 1)) if rows.n_st else np.zeros(M + 1, int)
    soft_st, r1_st, r2_st = (rows.soft[rows.n_in:], rows.rho1[rows.n_in:], rows.rho2[rows.n_in:])
    out = []
    for i in range(M):
        a, b = int(bounds[i]), int(bounds[i + 1])
        if b > a:
            cr, dr = C[a:b].copy(), d[a:b].copy()
        else:
            cr, dr = np.zeros((0, n0)), np.zeros(0)
        out.append(LocalCondensed(i, gu[i], gx[i], H[i], g[i], cr, dr, soft_st[a:b].copy(),
                                  r1_st[a:b].copy(), r2_st[a:b].copy(), _dev=(Hd, gd, i)))
    return out


def assemble_qp(spec, locals_) -> CondensedQp:
    """Sum the per-node cost contributions in ascending list order on the
    device (R-bar first, then each node's h, g; symmetrised) and stack the
    constraint rows: input rows first, then each node's block
    (``condensing.py:334-360``)."""
    N, nu = spec.horizon, spec.n_u
    n0 = N * nu
    cost = cost_to_standard_form(spec)
    rb = np.zeros((n0, n0))
    for k in range(N):
        rb[k * nu:(k + 1) * nu, k * nu:(k + 1) * nu] = cost.r_blocks[k]
    r_lin = cost.r_lin.reshape(-1)
    eng = _dev.engine(_qp_topo)
    locs = list(locals_)
    src = locs[0]._dev if locs and locs[0]._dev is not None else None
    same = src is not None and all(lc._dev is not None and lc._dev[0] is src[0]
                                   and lc._dev[2] == k for k, lc in enumerate(locs)) \
        and src[0].shape[0] == len(locs)
    if same and src[0].device == eng.device:
        Hs, gs = src[0], src[1]
    else:  # arbitrary LocalCondensed lists: upload their (h, g)
        Hs = eng.h2d(np.stack([np.asarray(lc.h, dtype=float) for lc in locs])
                     if locs else np.zeros((0, n0, n0)), np.float64)
        gs = eng.h2d(np.stack([np.asarray(lc.g, dtype=float) for lc in locs])
                     if locs else np.zeros((0, n0)), np.float64)
    H = eng.empty((n0, n0), np.float64)
    g = eng.empty((n0,), np.float64)
    count = len(locs)
    rbd, rld = eng.h2d(rb, np.float64), eng.h2d(r_lin, np.float64)
    eng.ctx.call("gm_sum_nodes", 1, count, n0 * n0, n0, Hs.data_ptr() if count else None,
                 rbd.data_ptr(), H.data_ptr(), eng.stream_ptr())
    eng.ctx.call("gm_sum_nodes", 1, count, n0, 0, gs.data_ptr() if count else None,
                 rld.data_ptr(), g.data_ptr(), eng.stream_ptr())
    rows = spec_rows(spec, spec.n_state, nu)
    cu = np.zeros((rows.n_in, n0))
    for r in range(rows.n_in):
        k = rows.in_stage[r]
        cu[r, k * nu:(k + 1) * nu] = rows.in_c[r]
    c_all = [cu] + [np.asarray(lc.c_rows, dtype=float).reshape(-1, n0) for lc in locs]
    d_all = [rows.in_d] + [np.asarray(lc.d_rows, dtype=float) for lc in locs]
    soft = [np.zeros(rows.n_in, dtype=bool)] + [np.asarray(lc.soft, dtype=bool) for lc in locs]
    rho1 = [np.zeros(rows.n_in)] + [np.asarray(lc.rho1, dtype=float) for lc in locs]
    rho2 = [np.zeros(rows.n_in)] + [np.asarray(lc.rho2, dtype=float) for lc in locs]
    return CondensedQp(h=H.cpu().numpy(), g=g.cpu().numpy(), c=np.vstack(c_all),
                       d=np.concatenate(d_all), soft=np.concatenate(soft),
                       rho1=np.concatenate(rho1), rho2=np.concatenate(rho2))
