"""CPU ORACLE for the GNN-MPC hot path -- TEST INFRASTRUCTURE, NOT PRODUCT.

A NumPy/SciPy restatement of the reference algorithm (arXiv 2602.17601,
package ``gnnmpc`` under ``/root/reference/pkg/src``).  Every function cites
the reference ``file:line`` it follows.  It exists for three consumers only:

* ``tests/``           -- the checker the CUDA path is compared against;
* ``__graft_entry__.smoke()`` -- one small parity check on ``cuda:0``;
* ``bench.py``         -- the ``cpu_baseline`` leg and ``--impl reference``.

The product package (``paper_2602_17601_b200``) never imports this module;
its GPU path fails loudly when the CUDA library is missing.

Parity pin: ``tests/test_oracle_golden.py`` checks this port against golden
vectors produced by the reference itself (``oracle/make_golden.py`` ->
``tests/golden/*.npz``).  The arithmetic follows the reference operation by
operation (same batched products, same reduction axes), so the two agree to
~1e-15 and run at comparable speed; the timing leg therefore stands in for
the reference's own CPU path on the GPU box, where ``/root/reference`` does
not exist.

All functions accept duck-typed objects: anything with the attributes of the
reference's ``GraphTopology`` / ``GnnModel`` / ``OcpSpec`` /
``LinearizedDynamics`` works, so the reference's own objects and the
product package's mirrors are interchangeable here.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from types import SimpleNamespace

import numpy as np
import scipy.linalg as sla

# QpStatus values, in the reference's declaration order (qpsolver.py:24-28)
OPTIMAL, MAX_ITERATIONS, PRIMAL_INFEASIBLE, NUMERICAL_FAILURE = (
    "optimal", "max_iterations", "primal_infeasible", "numerical_failure")


# --------------------------------------------------------------------------
# index construction (bit-exact targets)
# --------------------------------------------------------------------------

def edge_lists(topo):
    """dst, src and the padded in-edge gather table (gnn.py:107-126).

    gather[i, s] = position of node i's s-th in-edge in the canonical edge
    list, padded with E (a phantom zero-message row)."""
    M = topo.node_count
    dst_l, src_l = [], []
    for i, ns in enumerate(topo.in_neighbors):
        for j in ns:
            dst_l.append(i)
            src_l.append(j)
    E = len(dst_l)
    width = max(1, max((len(ns) for ns in topo.in_neighbors), default=0))
    gather = np.full((M, width), E, dtype=np.intp)
    pos = 0
    for i, ns in enumerate(topo.in_neighbors):
        gather[i, : len(ns)] = np.arange(pos, pos + len(ns))
        pos += len(ns)
    return np.array(dst_l, dtype=np.intp), np.array(src_l, dtype=np.intp), gather


def slot_tables(topo):
    """Closed-neighbourhood ELL table (condensing.py:158-172): slot 0 is the
    node, pad = M (phantom zero node); edge_slot[e] = slot of edge e."""
    M = topo.node_count
    S = 1 + max((len(ns) for ns in topo.in_neighbors), default=0)
    nbr_idx = np.full((M, S), M, dtype=np.intp)
    nbr_idx[:, 0] = np.arange(M)
    slots = []
    for i, ns in enumerate(topo.in_neighbors):
        nbr_idx[i, 1 : 1 + len(ns)] = ns
        slots.extend(range(1, 1 + len(ns)))
    return nbr_idx, np.array(slots, dtype=np.intp)


# --------------------------------------------------------------------------
# MLP primitives (mlp.py)
# --------------------------------------------------------------------------

def mlp_apply(params, x, keep_pre=False):
    """Batched forward (mlp.py:81-107); optionally return pre-activations."""
    pres = []
    h = x
    n = len(params.weights)
    for l in range(n):
        z = h @ params.weights[l].T + params.biases[l]
        pres.append(z)
        h = np.maximum(z, 0.0) if l < n - 1 else z
    return (h, pres) if keep_pre else h


def mlp_input_jacobian(params, x):
    """d out / d in accumulated from the output side (mlp.py:132-145);
    ReLU derivative at exactly 0 is 0 (strict > 0 mask)."""
    _, pres = mlp_apply(params, x, keep_pre=True)
    lead = x.shape[:-1]
    J = np.broadcast_to(params.weights[-1], lead + params.weights[-1].shape)
    for l in range(len(params.weights) - 2, -1, -1):
        J = (J * (pres[l] > 0.0)[..., None, :]) @ params.weights[l]
    return np.ascontiguousarray(J)


# --------------------------------------------------------------------------
# GNN dynamics and its linearisation (gnn.py)
# --------------------------------------------------------------------------

def _forward_parts(model, topo, X, U):
    """Normalised edge features, aggregated messages, phi input and output
    (gnn.py:129-150)."""
    nrm = model.normalization
    dst, src, gather = edge_lists(topo)
    Hn = (X - nrm.state_mean) / nrm.state_scale
    ef = (X[..., dst, :] - X[..., src, :]) / nrm.state_scale
    if dst.size:
        msg = mlp_apply(model.psi, ef)
        pad = np.zeros(msg.shape[:-2] + (1, model.n_m))
        agg = np.concatenate([msg, pad], axis=-2)[..., gather, :].sum(axis=-2)
    else:
        agg = np.zeros(X.shape[:-1] + (model.n_m,))
    Un = (U - nrm.input_mean) / nrm.input_scale
    Ub = np.broadcast_to(Un[..., None, :], X.shape[:-1] + (model.n_u,))
    z = np.concatenate([Hn, agg, Ub], axis=-1)
    return ef, agg, z, mlp_apply(model.phi, z)


# --------------------------------------------------------------------------
# training gradients (training.py:99-150)
# --------------------------------------------------------------------------

def _mlp_backward(params, x, g_out):
    """Reverse mode of mlp_apply (mlp.py:110-129): weight / bias gradients
    summed over the batch and the input gradient."""
    _, pres = mlp_apply(params, x, keep_pre=True)
    n = len(params.weights)
    acts = [x] + [np.maximum(z, 0.0) for z in pres[:-1]]
    gw, gb = [None] * n, [None] * n
    g = g_out
    for l in range(n - 1, -1, -1):
        if l != n - 1:
            g = g * (pres[l] > 0.0)
        gf = g.reshape(-1, g.shape[-1])
        gw[l] = gf.T @ acts[l].reshape(-1, acts[l].shape[-1])
        gb[l] = gf.sum(axis=0)
        g = g @ params.weights[l]
    return gw, gb, g


def loss_gradients(model, topo, X, U, Xn, weights, l2_lambda):
    """Batch loss sum(W r^2)/B + lambda |p|^2 and its gradient, order psi W,
    psi b, phi W, phi b (training.py:99-150)."""
    B, n_p = X.shape[0], model.n_p
    dst, src, gather = edge_lists(topo)
    ef, agg, z, dv = _forward_parts(model, topo, X, U)
    v1 = X[..., n_p:] + dv
    p1 = X[..., :n_p] + model.dt * v1
    r = np.concatenate([p1, v1], axis=-1) - Xn
    loss = float(np.sum(weights * r * r) / B)
    gp = 2.0 * weights * r / B
    g_dv = gp[..., n_p:] + model.dt * gp[..., :n_p]
    gw_phi, gb_phi, g_z = _mlp_backward(model.phi, z, g_dv)
    if dst.size:
        nx = X.shape[-1]
        g_msg = g_z[..., nx:nx + model.n_m][..., dst, :]
        gw_psi, gb_psi, _ = _mlp_backward(model.psi, ef, g_msg)
    else:
        gw_psi = [np.zeros_like(W) for W in model.psi.weights]
        gb_psi = [np.zeros_like(b) for b in model.psi.biases]
    grads = gw_psi + gb_psi + gw_phi + gb_phi
    if l2_lambda > 0:
        params = model.psi.weights + model.psi.biases + model.phi.weights + model.phi.biases
        grads = [g + 2.0 * l2_lambda * p for g, p in zip(grads, params)]
        loss += l2_lambda * sum(float(np.sum(p * p)) for p in params)
    return loss, grads


def step_array(model, topo, X, U):
    """One model step, velocity first then position (gnn.py:153-159)."""
    n_p = model.n_p
    _, _, _, dv = _forward_parts(model, topo, X, U)
    v1 = X[..., n_p:] + dv
    p1 = X[..., :n_p] + model.dt * v1
    return np.concatenate([p1, v1], axis=-1)


def linearize(model, topo, X, U):
    """Exact per-stage Jacobian blocks and affine offsets (gnn.py:237-298).

    X: (K, M, nx), U: (K, nu).  Returns a namespace with a_self (K,M,nx,nx),
    a_nbr (K,E,nx,nx) in topo.edges order, b (K,M,nx,nu), c (K,M,nx)."""
    K, M, nx = X.shape
    n_p, n_m = model.n_p, model.n_m
    nrm = model.normalization
    dst, src, gather = edge_lists(topo)
    E = dst.size
    ef, _, z, _ = _forward_parts(model, topo, X, U)
    Jphi = mlp_input_jacobian(model.phi, z)  # (K, M, n_p, nx + n_m + n_u)
    Jh, Jm, Ju = Jphi[..., :nx], Jphi[..., nx : nx + n_m], Jphi[..., nx + n_m :]
    inv_sx = 1.0 / nrm.state_scale
    inv_su = 1.0 / nrm.input_scale
    if E:
        Jpsi = mlp_input_jacobian(model.psi, ef)  # (K, E, n_m, nx)
        Jpsi_pad = np.concatenate([Jpsi, np.zeros((K, 1, n_m, nx))], axis=1)
        Jpsi_node = Jpsi_pad[:, gather].sum(axis=2)  # (K, M, n_m, nx)
        dself = (Jh + Jm @ Jpsi_node) * inv_sx
        dnbr = -(Jm[:, dst] @ Jpsi) * inv_sx
    else:
        dself = Jh * inv_sx
        dnbr = np.zeros((K, 0, n_p, nx))
    du = Ju * inv_su
    vel_sel = np.zeros((n_p, nx))
    vel_sel[:, n_p:] = np.eye(n_p)
    dvdx = dself + vel_sel
    a_self = np.zeros((K, M, nx, nx))
    a_self[..., :n_p, :n_p] = np.eye(n_p)
    a_self[..., :n_p, :] += model.dt * dvdx
    a_self[..., n_p:, :] = dvdx
    a_nbr = np.zeros((K, E, nx, nx))
    a_nbr[..., :n_p, :] = model.dt * dnbr
    a_nbr[..., n_p:, :] = dnbr
    b = np.zeros((K, M, nx, model.n_u))
    b[..., :n_p, :] = model.dt * du
    b[..., n_p:, :] = du
    f = step_array(model, topo, X, U)
    c = f - (a_self @ X[..., None])[..., 0] - (b @ U[:, None, :, None])[..., 0]
    if E:
        contrib = (a_nbr @ X[:, src, :, None])[..., 0]
        acc = np.zeros((K, M, nx))
        np.add.at(acc, (slice(None), dst), contrib)
        c -= acc
    return SimpleNamespace(topology=topo, horizon=K, a_self=a_self, a_nbr=a_nbr, b=b, c=c,
                           n_state=nx, n_u=model.n_u)


def linearize_trajectory(model, topo, states, inputs):
    """First N states of an (N or N+1)-state nominal trajectory (gnn.py:308-321)."""
    inputs = np.asarray(inputs, dtype=float)
    states = np.asarray(states, dtype=float)
    N = inputs.shape[0]
    if states.shape[0] not in (N, N + 1):
        raise ValueError("need one linearization state per stage")
    return linearize(model, topo, states[:N], inputs)


# --------------------------------------------------------------------------
# condensing (condensing.py)
# --------------------------------------------------------------------------

def _pad_blocks(lin):
    """a_pad (N, M, S, nx, nx): slot-0 self block, edge blocks scattered to
    their slots (condensing.py:173-179)."""
    topo = lin.topology
    nbr_idx, edge_slot = slot_tables(topo)
    N, M, nx, _ = lin.a_self.shape
    a_pad = np.zeros((N, M, nbr_idx.shape[1], nx, nx))
    a_pad[:, :, 0] = lin.a_self
    if edge_slot.size:
        dst, _, _ = edge_lists(topo)
        a_pad[:, dst, edge_slot] = lin.a_nbr
    return nbr_idx, a_pad


def condense_gammas(lin, x0, threads=1):
    """Stage-by-stage neighbourhood recursion on [Gamma_x | Gamma_u]
    (condensing.py:182-228).  Returns (gamma_u (M,N+1,nx,N*nu),
    gamma_x (M,N+1,nx))."""
    M = lin.topology.node_count
    N = lin.horizon
    nx, nu = lin.a_self.shape[-1], lin.b.shape[-1]
    nbr_idx, a_pad = _pad_blocks(lin)
    work = np.zeros((M + 1, N + 1, nx, 1 + N * nu))
    work[:M, 0, :, 0] = np.asarray(x0, dtype=float).reshape(M, nx)
    parts = np.array_split(np.arange(M), threads) if threads > 1 else [np.arange(M)]

    def advance(rows, n):
        live = 1 + n * nu
        nb = work[:, n, :, :live][nbr_idx[rows]]
        nxt = (a_pad[n, rows] @ nb).sum(axis=1)
        nxt[..., 0] += lin.c[n, rows]
        work[rows, n + 1, :, :live] = nxt
        work[rows, n + 1, :, live : live + nu] = lin.b[n, rows]

    pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    try:
        for n in range(N):
            if pool is None:
                advance(parts[0], n)
            else:
                list(pool.map(lambda r, n=n: advance(r, n), parts))
    finally:
        if pool is not None:
            pool.shutdown()
    return work[:M, :, :, 1:], work[:M, :, :, 0]


def standard_form(spec):
    """q_lin = -2 Q x_ref, r_lin = -2 R u_ref (condensing.py:152-155)."""
    q_lin = -2.0 * np.einsum("mkab,mkb->mka", spec.q, spec.x_ref)
    r_lin = -2.0 * np.einsum("kab,kb->ka", spec.r, spec.u_ref)
    return q_lin, r_lin


def r_bar(spec):
    """Block-diagonal input Hessian and stacked linear term (condensing.py:326-331)."""
    N, nu = spec.r.shape[0], spec.r.shape[-1]
    rb = np.zeros((N * nu, N * nu))
    for k in range(N):
        rb[k * nu : (k + 1) * nu, k * nu : (k + 1) * nu] = spec.r[k]
    return rb, standard_form(spec)[1].reshape(-1)


def input_rows(spec):
    """Stage-major input constraint rows in block k (condensing.py:312-323)."""
    N, nu = spec.horizon, spec.r.shape[-1]
    if spec.input_constraints is None:
        return np.zeros((0, N * nu)), np.zeros(0)
    Cs, ds = [], []
    for k, (Ck, dk) in enumerate(spec.input_constraints):
        Ck = np.atleast_2d(np.asarray(Ck, dtype=float))
        row = np.zeros((Ck.shape[0], N * nu))
        row[:, k * nu : (k + 1) * nu] = Ck
        Cs.append(row)
        ds.append(np.atleast_1d(np.asarray(dk, dtype=float)))
    return np.vstack(Cs), np.concatenate(ds)


def node_rows(spec, i, gu_i, gx_i, n_cols):
    """State constraints of node i mapped into input space, stage ascending
    (condensing.py:263-282)."""
    mine = sorted((s for s in spec.state_constraints if s.node == i), key=lambda s: s.stage)
    if not mine:
        return (np.zeros((0, n_cols)), np.zeros(0), np.zeros(0, dtype=bool), np.zeros(0),
                np.zeros(0))
    C, d, soft, r1, r2 = [], [], [], [], []
    for sc in mine:
        cc = np.atleast_2d(np.asarray(sc.c, dtype=float))
        C.append(cc @ gu_i[sc.stage])
        d.append(np.atleast_1d(np.asarray(sc.d, dtype=float)) - cc @ gx_i[sc.stage])
        rows = cc.shape[0]
        soft += [bool(sc.soft)] * rows
        r1 += [float(sc.rho1)] * rows
        r2 += [float(sc.rho2)] * rows
    return (np.vstack(C), np.concatenate(d), np.array(soft, dtype=bool), np.array(r1),
            np.array(r2))


def condense_ocp(spec, lin, x0, threads=1, gammas=None):
    """Fused stage-wise H/g accumulation plus constraint stacking
    (condensing.py:363-406).  Objective u'Hu + g'u (no 1/2)."""
    M = spec.topology.node_count
    N, nu = spec.horizon, spec.r.shape[-1]
    q_lin, _ = standard_form(spec)
    gu, gx = gammas if gammas is not None else condense_gammas(lin, x0, threads=threads)
    H, g = r_bar(spec)
    g = g.copy()
    for k in range(1, N + 1):
        w = min(k, N) * nu
        Gk = gu[:, k, :, :w]
        QG = spec.q[:, k] @ Gk
        H[:w, :w] += np.tensordot(Gk, QG, axes=([0, 1], [0, 1]))
        wk = 2.0 * (spec.q[:, k] @ gx[:, k, :, None])[..., 0] + q_lin[:, k]
        g[:w] += np.einsum("mab,ma->b", Gk, wk)
    cu, du = input_rows(spec)
    Cs, ds = [cu], [du]
    soft = [np.zeros(cu.shape[0], dtype=bool)]
    r1 = [np.zeros(cu.shape[0])]
    r2 = [np.zeros(cu.shape[0])]
    for i in range(M):
        a, b_, s_, p1, p2 = node_rows(spec, i, gu[i], gx[i], N * nu)
        Cs.append(a)
        ds.append(b_)
        soft.append(s_)
        r1.append(p1)
        r2.append(p2)
    return SimpleNamespace(h=0.5 * (H + H.T), g=g, c=np.vstack(Cs), d=np.concatenate(ds),
                           soft=np.concatenate(soft), rho1=np.concatenate(r1),
                           rho2=np.concatenate(r2))


def local_hessian_gradient(gamma_u, gamma_x, q_blocks, q_lin):
    """One node's symmetrised Hessian and gradient (condensing.py:231-243):
    h = sum_k Gu_k' Q_k Gu_k over all N+1 stages, g = sum_k Gu_k' w_k with
    w_k = 2 Q_k Gx_k + q_lin_k."""
    h = np.zeros((gamma_u.shape[-1],) * 2)
    g = np.zeros(gamma_u.shape[-1])
    for k in range(gamma_u.shape[0]):
        G = gamma_u[k]
        h += G.T @ (q_blocks[k] @ G)
        g += G.T @ (2.0 * q_blocks[k] @ gamma_x[k] + q_lin[k])
    return 0.5 * (h + h.T), g


def condense_local(spec, lin, x0):
    """Per-node (node, h, g, rows) after the recursion (condensing.py:285-295)."""
    q_lin, _ = standard_form(spec)
    gu, gx = condense_gammas(lin, x0)
    n_cols = spec.horizon * spec.r.shape[-1]
    out = []
    for i in range(spec.topology.node_count):
        h, g = local_hessian_gradient(gu[i], gx[i], spec.q[i], q_lin[i])
        rows = node_rows(spec, i, gu[i], gx[i], n_cols)
        out.append(SimpleNamespace(node=i, gamma_u=gu[i], gamma_x=gx[i], h=h, g=g, c_rows=rows[0],
                                   d_rows=rows[1], soft=rows[2], rho1=rows[3], rho2=rows[4]))
    return out


def assemble_qp(spec, locals_):
    """R-bar plus the node contributions in list order, symmetrised; input
    rows then each node's rows (condensing.py:334-360)."""
    H, g = r_bar(spec)
    g = g.copy()
    for lc in locals_:
        H = H + lc.h
        g = g + lc.g
    cu, du = input_rows(spec)
    return SimpleNamespace(
        h=0.5 * (H + H.T), g=g, c=np.vstack([cu] + [lc.c_rows for lc in locals_]),
        d=np.concatenate([du] + [lc.d_rows for lc in locals_]),
        soft=np.concatenate([np.zeros(cu.shape[0], dtype=bool)] + [lc.soft for lc in locals_]),
        rho1=np.concatenate([np.zeros(cu.shape[0])] + [lc.rho1 for lc in locals_]),
        rho2=np.concatenate([np.zeros(cu.shape[0])] + [lc.rho2 for lc in locals_]))


def expand_soft_constraints(qp):
    """One penalised slack per soft row (condensing.py:419-439).
    Returns (H, g, C, d, n_original)."""
    idx = np.flatnonzero(qp.soft)
    n = qp.h.shape[0]
    if idx.size == 0:
        return qp.h, qp.g, qp.c, qp.d, n
    ns = idx.size
    m0 = qp.c.shape[0]
    H = np.zeros((n + ns, n + ns))
    H[:n, :n] = qp.h
    H[n:, n:] = np.diag(qp.rho2[idx])
    g = np.concatenate([qp.g, qp.rho1[idx]])
    C = np.zeros((m0 + ns, n + ns))
    C[:m0, :n] = qp.c
    C[idx, n + np.arange(ns)] = -1.0
    C[m0 + np.arange(ns), n + np.arange(ns)] = -1.0
    return H, g, C, np.concatenate([qp.d, np.zeros(ns)]), n


def reconstruct_states(gamma_u, gamma_x, u):
    """x^i = Gamma_u^i u + Gamma_x^i (condensing.py:409-416)."""
    return gamma_u @ np.asarray(u, dtype=float).reshape(-1) + gamma_x


# --------------------------------------------------------------------------
# dense QP interior point (qpsolver.py)
# --------------------------------------------------------------------------

def _step_to_boundary(x, dx):
    """Largest a in [0,1] with x + a dx > 0 (qpsolver.py:238-243)."""
    neg = dx < 0
    if not np.any(neg):
        return 1.0
    return float(min(1.0, np.min(-x[neg] / dx[neg])))


def _classify_rows(C):
    """Single-nonzero rows (diagonal Schur contribution) vs general rows
    (qpsolver.py:100-109)."""
    nz = C != 0.0
    cnt = nz.sum(axis=1)
    single = np.flatnonzero(cnt == 1)
    general = np.flatnonzero(cnt != 1)
    cols = nz[single].argmax(axis=1) if single.size else np.zeros(0, dtype=np.intp)
    vals = C[single, cols] if single.size else np.zeros(0)
    return single, cols, vals, general


def _kkt_residuals(H, g, C, d, u, lam):
    """(stationarity, primal infeasibility, complementarity) (qpsolver.py:90-97)."""
    m = d.shape[0]
    if m:
        r_stat = float(np.max(np.abs(2.0 * H @ u + g + C.T @ lam)))
        viol = C @ u - d
        return r_stat, float(max(0.0, np.max(viol))), float(np.max(np.abs(lam * viol)))
    return float(np.max(np.abs(2.0 * H @ u + g))), 0.0, 0.0


def solve_qp(H, g, C, d, tolerance=1e-8, max_iterations=50, regularization=1e-9,
             fraction_to_boundary=0.995, warm_start=None):
    """Mehrotra predictor-corrector for min u'Hu + g'u s.t. Cu <= d
    (qpsolver.py:112-235).  Returns a namespace mirroring QpSolution with
    ``status`` as the QpStatus value string."""
    H = np.asarray(H, dtype=float)
    g = np.asarray(g, dtype=float).reshape(-1)
    n = g.shape[0]
    C = np.asarray(C, dtype=float).reshape(-1, n) if np.size(C) else np.zeros((0, n))
    d = np.asarray(d, dtype=float).reshape(-1)
    m = d.shape[0]
    tol = tolerance

    def result(u, lam, status, it, rs, rp, rc):
        return SimpleNamespace(u=u, duals=lam, status=status, iterations=it, stationarity=rs,
                               primal_infeas=rp, complementarity=rc)

    g_inf = float(np.max(np.abs(g))) if n else 0.0
    scale_k = min(1.0, max(float(np.max(np.abs(H))) if n else 0.0, g_inf))
    scale_g = scale_k + g_inf
    comp_ref = scale_k
    H2 = 2.0 * H + regularization * np.eye(n)

    if m == 0:  # qpsolver.py:131-144
        factor = None
        for boost in (0.0, regularization, regularization * 1e3, regularization * 1e6):
            try:
                factor = sla.cho_factor(2.0 * H + boost * np.eye(n), lower=True,
                                        check_finite=False)
                break
            except np.linalg.LinAlgError:
                continue
        if factor is None:
            return result(np.zeros(n), np.zeros(0), NUMERICAL_FAILURE, 0, np.inf, np.inf, np.inf)
        u = sla.cho_solve(factor, -g, check_finite=False)
        rs, rp, rc = _kkt_residuals(H, g, C, d, u, np.zeros(0))
        return result(u, np.zeros(0), OPTIMAL, 0, rs, rp, rc)

    u = np.zeros(n) if warm_start is None else np.asarray(warm_start, dtype=float).copy()
    if u.shape != (n,):
        raise ValueError("warm start dimension mismatch")
    slack = np.maximum(d - C @ u, 1.0) * 1.1
    lam = np.ones(m)
    single, s_cols, s_vals, general = _classify_rows(C)
    Cg = C[general]
    best = [np.inf, None]

    def track(u, lam):
        rs, rp, rc = _kkt_residuals(H, g, C, d, u, lam)
        merit = max(rs / scale_g, rp, rc / max(comp_ref, 1e-300))
        if merit < best[0]:
            best[0] = merit
            best[1] = (u.copy(), lam.copy(), rs, rp, rc)
        return rs, rp, rc

    def from_best(status, it):
        ub, lb, rs, rp, rc = best[1]
        return result(ub, lb, status, it, rs, rp, rc)

    K = np.empty_like(H2)
    for it in range(max_iterations):
        rs, rp, rc = track(u, lam)
        if rs <= tol * scale_g and rp <= tol and rc <= tol * comp_ref:
            return result(u, lam, OPTIMAL, it, rs, rp, rc)
        if np.max(lam) > 1e12 and rp > 1e-6:
            return from_best(PRIMAL_INFEASIBLE, it)
        w = lam / slack
        np.copyto(K, H2)
        diag = np.einsum("ii->i", K)
        if single.size:
            diag += np.bincount(s_cols, weights=w[single] * s_vals * s_vals, minlength=n)
        if general.size:
            K += (Cg * w[general, None]).T @ Cg
        factor, boost = None, 0.0
        for _ in range(4):  # escalating static regularisation, qpsolver.py:186-198
            try:
                factor = sla.cho_factor(K, lower=True, check_finite=False)
                break
            except np.linalg.LinAlgError:
                bump = max(regularization * 1e3, 1e-12) if boost == 0.0 else boost * 1e3
                diag += bump - boost
                boost = bump
        if factor is None:
            return from_best(NUMERICAL_FAILURE, it)
        r_dual = 2.0 * H @ u + g + C.T @ lam
        r_pri = C @ u + slack - d
        mu = float(lam @ slack) / m

        def direction(rc_vec):
            rhs = -r_dual - C.T @ ((rc_vec + lam * r_pri) / slack)
            du = sla.cho_solve(factor, rhs, check_finite=False)
            ds = -r_pri - C @ du
            return du, (rc_vec - lam * ds) / slack, ds

        du_a, dl_a, ds_a = direction(-lam * slack)
        ap = _step_to_boundary(slack, ds_a)
        ad = _step_to_boundary(lam, dl_a)
        mu_aff = float((lam + ad * dl_a) @ (slack + ap * ds_a)) / m
        sigma = (mu_aff / mu) ** 3 if mu > 0 else 0.0
        du, dl, ds = direction(-lam * slack - dl_a * ds_a + sigma * mu)
        alpha = min(fraction_to_boundary * _step_to_boundary(slack, ds),
                    fraction_to_boundary * _step_to_boundary(lam, dl))
        u = u + alpha * du
        slack = slack + alpha * ds
        lam = lam + alpha * dl
        if not (np.all(np.isfinite(u)) and np.all(np.isfinite(lam))
                and np.all(np.isfinite(slack))):
            return from_best(NUMERICAL_FAILURE, it + 1)
    rs, rp, rc = track(u, lam)
    if rs <= tol * scale_g and rp <= tol and rc <= tol * comp_ref:
        return result(u, lam, OPTIMAL, max_iterations, rs, rp, rc)
    return from_best(MAX_ITERATIONS, max_iterations)


# --------------------------------------------------------------------------
# receding-horizon step (mpc.py)
# --------------------------------------------------------------------------

def shift(states, inputs):
    """Advance one stage, duplicating the terminal entries (mpc.py:90-99)."""
    s = np.empty_like(states)
    s[:-1] = states[1:]
    s[-1] = states[-1]
    u = np.empty_like(inputs)
    if inputs.shape[0] > 1:
        u[:-1] = inputs[1:]
    u[-1] = inputs[-1]
    return s, u


def mpc_step(model, topo, spec, x_measured, lin_states, lin_inputs, horizon, warm_start=True,
             solver=None, sqp_iterations=1, sqp_damping=1.0, threads=1, fallback="hold-previous-input",
             last_applied=None, timings=None, input_filter_tau=None, filtered_input=None, dt=None):
    """One RTI control step (mpc.py:102-200), state passed as plain arrays.

    Returns dict(u_applied, lin_states, lin_inputs, planned_states,
    planned_inputs, status, iterations).  ``timings`` (a dict) receives
    per-phase wall-clock milliseconds in the reference's StepTiming buckets."""
    import time

    solver = dict(solver or {})
    N = horizon
    x_meas = np.asarray(x_measured, dtype=float)
    n_u = lin_inputs.shape[1]
    ls = np.array(lin_states, dtype=float, copy=True)
    li = np.array(lin_inputs, dtype=float, copy=True)
    ls[0] = x_meas
    status, iters, solved = None, 0, False
    tm = {"linearize_ms": 0.0, "condense_ms": 0.0, "solve_ms": 0.0}
    for _ in range(sqp_iterations):
        t0 = time.perf_counter()
        lin = linearize_trajectory(model, topo, ls[:N], li)
        t1 = time.perf_counter()
        gam = condense_gammas(lin, x_meas, threads=threads)
        qp = condense_ocp(spec, lin, x_meas, threads=threads, gammas=gam)
        H, g, C, d, _ = expand_soft_constraints(qp)
        t2 = time.perf_counter()
        warm = None
        if warm_start:
            warm = np.zeros(H.shape[0])
            warm[: N * n_u] = li.reshape(-1)
        sol = solve_qp(H, g, C, d, warm_start=warm, **solver)
        t3 = time.perf_counter()
        tm["linearize_ms"] += (t1 - t0) * 1e3
        tm["condense_ms"] += (t2 - t1) * 1e3
        tm["solve_ms"] += (t3 - t2) * 1e3
        status = sol.status
        iters += sol.iterations
        if status in (OPTIMAL, MAX_ITERATIONS):
            uf = sol.u[: N * n_u]
            plan = reconstruct_states(gam[0], gam[1], uf)
            a = sqp_damping
            ls = (1 - a) * ls + a * plan.transpose(1, 0, 2)
            li = (1 - a) * li + a * uf.reshape(N, n_u)
            solved = True
        else:
            solved = False
            break
    if solved:
        u_app = li[0].copy()
    else:
        u_app = (np.array(last_applied, dtype=float) if
                 (fallback == "hold-previous-input" and last_applied is not None)
                 else np.zeros(n_u))
        ls = np.array(lin_states, dtype=float, copy=True)
        ls[0] = x_meas
        li = np.array(lin_inputs, dtype=float, copy=True)
    planned_states = ls.transpose(1, 0, 2).copy()
    planned_inputs = li.copy()
    filtered = filtered_input
    if input_filter_tau is not None:  # first-order input smoothing (mpc.py:178-183)
        alpha = dt / (input_filter_tau + dt)
        prev = np.asarray(filtered, dtype=float) if filtered is not None else u_app
        u_app = prev + alpha * (u_app - prev)
        filtered = u_app.copy()
    ns, ni = shift(ls, li)
    if timings is not None:
        timings.update(tm)
    return dict(u_applied=u_app, lin_states=ns, lin_inputs=ni, planned_states=planned_states,
                planned_inputs=planned_inputs, status=status, iterations=iters,
                filtered_input=filtered)


# --------------------------------------------------------------------------
# chain plant (trunk.py) and closed-loop tracking (experiments.py, mpc.py)
# -- the environment of BASELINE cfg2, used to check the device closed loop
# --------------------------------------------------------------------------

def trunk_params(node_count, node_mass=0.08, coupling_stiffness=300.0, coupling_damping=2.0,
                 bend_stiffness=25.0, rest_length=0.15, gravity=(0.0, 0.0, -9.81), u_max=8.0,
                 dt_sim=1e-3, dt=0.01):
    """ChainConfig defaults (trunk.py:23-73) as a dict; six horizontal tendons
    60 degrees apart, each attached to every moving node (trunk.py:51-61)."""
    angles = np.deg2rad([0, 60, 120, 180, 240, 300])
    dirs = np.stack([np.cos(angles), np.sin(angles), np.zeros(6)], axis=1)
    M = node_count
    fmap = np.zeros((M, 3, 6))
    for t in range(6):  # tendon_force_map (trunk.py:96-104)
        for i in range(1, M):
            fmap[i, :, t] = (1.0 / (M - 1)) * dirs[t]
    rest = np.zeros((M, 3))
    rest[:, 2] = -rest_length * np.arange(M)
    return dict(M=M, m=node_mass, k=coupling_stiffness, c=coupling_damping, kb=bend_stiffness,
                L=rest_length, g=np.asarray(gravity, dtype=float), u_max=u_max, dt_sim=dt_sim, dt=dt,
                substeps=int(round(dt / dt_sim)), fmap=fmap, rest=rest)


def trunk_accelerations(P, p, v, u):
    """Net force / mass (trunk.py:116-135)."""
    f = np.broadcast_to(P["m"] * P["g"], p.shape).copy()
    delta = p[1:] - p[:-1]
    length = np.maximum(np.linalg.norm(delta, axis=-1, keepdims=True), 1e-12)
    axial = P["k"] * (length - P["L"]) * (delta / length)
    damp = P["c"] * (v[1:] - v[:-1])
    f[1:] -= axial + damp
    f[:-1] += axial + damp
    f[1:] -= P["kb"] * (p[1:] - P["rest"][1:])
    f += P["fmap"] @ u
    return f / P["m"]


def trunk_step(P, arr, u, clip_inputs=True):
    """step_state_array (trunk.py:148-160) for one (M, 6) state."""
    u = np.asarray(u, dtype=float)
    if clip_inputs:
        u = np.clip(u, 0.0, P["u_max"])
    p = arr[:, :3].copy()
    v = arr[:, 3:].copy()
    for _ in range(P["substeps"]):
        a = trunk_accelerations(P, p, v, u)
        v = v + P["dt_sim"] * a
        v[0] = 0.0
        p = p + P["dt_sim"] * v
        p[0] = P["rest"][0]
    return np.concatenate([p, v], axis=-1)


def circle_ref(radius, period, center):
    """references.py:12-30."""
    center = np.asarray(center, dtype=float)
    om = 2.0 * np.pi / period

    def ref(t):
        ang = om * np.asarray(t, dtype=float)
        pos = np.stack([radius * np.cos(ang), radius * np.sin(ang), np.zeros_like(ang)], -1) + center
        vel = np.stack([-radius * om * np.sin(ang), radius * om * np.cos(ang), np.zeros_like(ang)], -1)
        return pos, vel

    return ref


class _Spec:
    """Plain OCP container with the fields condense_ocp reads."""

    def __init__(self, topology, horizon, q, x_ref, r, u_ref, input_constraints, state_constraints):
        self.topology, self.horizon = topology, horizon
        self.q, self.x_ref, self.r, self.u_ref = q, x_ref, r, u_ref
        self.input_constraints, self.state_constraints = input_constraints, state_constraints


def tracking_specs(topo, horizon, dt, rest_arr, ref, n_u, u_max, q_pos=(500.0, 500.0, 100.0),
                   q_vel=(0.5, 0.5, 0.5), r_diag=2e-4):
    """tracking_spec_provider (experiments.py:107-139) with default
    TrackingWeights (experiments.py:90-104): t -> spec."""
    M, N = topo.node_count, horizon
    target = M - 1
    q = np.zeros((M, N + 1, 6, 6))
    q[target, :] = np.diag(np.concatenate([q_pos, q_vel]))
    r = np.tile(np.eye(n_u) * r_diag, (N, 1, 1))
    u_ref = np.zeros((N, n_u))
    box = (np.vstack([np.eye(n_u), -np.eye(n_u)]), np.concatenate([np.full(n_u, u_max), np.zeros(n_u)]))
    x_base = np.tile(rest_arr[:, None, :], (1, N + 1, 1))
    offs = np.arange(N + 1) * dt

    def spec(t):
        x_ref = x_base.copy()
        pos, vel = ref(t * dt + offs)
        x_ref[target, :, :3] = pos
        x_ref[target, :, 3:] = vel
        return _Spec(topo, N, q, x_ref, r, u_ref, [box] * N, [])

    return spec


def closed_loop(model, topo, P, specs, x0, n_steps, horizon):
    """run_closed_loop (mpc.py:224-264) with the chain plant; returns states
    (n_steps+1, M, 6), inputs (n_steps, n_u), statuses, iterations."""
    n_u = 6
    ls = np.tile(x0, (horizon + 1, 1, 1))
    li = np.zeros((horizon, n_u))
    x = np.array(x0, dtype=float)
    states, inputs, statuses, iters = [x.copy()], [], [], []
    last = None
    for t in range(n_steps):
        res = mpc_step(model, topo, specs(t), x, ls, li, horizon, last_applied=last)
        ls, li, last = res["lin_states"], res["lin_inputs"], res["u_applied"]
        inputs.append(res["u_applied"])
        statuses.append(res["status"])
        iters.append(res["iterations"])
        x = trunk_step(P, x, res["u_applied"])
        states.append(x.copy())
    return np.stack(states), np.stack(inputs), statuses, np.asarray(iters)
