"""Node-partitioned condensing for graphs too large for one device (cfg5).

The horizon recursion is sequential in the stage index but node-parallel
within a stage (condensing.py:211-224): node i at stage n+1 reads
only the stage-n rows of its closed neighbourhood.  With the nodes split into
contiguous id ranges (row slabs of the 2-D mesh), a rank owns rows
[lo, hi) of every per-node array and needs, per stage, only the stage-n Gamma
rows of its *halo* -- the in-neighbours of owned nodes that other ranks own.

Per RTI step:

1. K-LIN on owned nodes (the linearisation trajectory is replicated, so halo
   states are local);
2. per stage: K-REC on owned nodes, then one grouped point-to-point exchange
   of the boundary Gamma rows (torch.distributed batch_isend_irecv: NCCL over
   NVLink on GPUs, gloo on CPU);
3. K-HG partial over owned nodes (rank 0 adds R-bar / r_lin), all-reduce(sum)
   of H and g; state-constraint rows are computed by the owner of their node
   and all-reduced (every other rank contributes zeros);
4. the small QP is solved redundantly on every rank (identical inputs and a
   deterministic kernel give identical outputs: no broadcast needed);
5. the planned trajectory slice of owned nodes is all-gathered.

The exchange / reduction logic is plain torch.distributed, so the same code
runs the CPU (gloo) tests and the GPU (NCCL) path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .batch import shard_range
from .device import topology_csr


@dataclass
class NodePartition:
    world: int
    rank: int
    lo: int
    hi: int
    owner: np.ndarray          # (M,) rank owning each node
    halo: dict                 # peer rank -> node ids this rank receives (ascending)
    send: dict                 # peer rank -> node ids this rank sends (ascending)

    @property
    def owned(self) -> np.ndarray:
        return np.arange(self.lo, self.hi)


def partition_nodes(topo, world: int, rank: int) -> NodePartition:
    """Contiguous id ranges; halo = in-neighbours of owned nodes owned elsewhere."""
    M = topo.node_count
    bounds = [shard_range(M, world, r) for r in range(world)]
    owner = np.empty(M, dtype=np.int64)
    for r, (a, b) in enumerate(bounds):
        owner[a:b] = r
    ptr, src = topology_csr(topo)

    def needs_of(r):
        a, b = bounds[r]
        nb = np.unique(src[ptr[a]:ptr[b]])
        return nb[(nb < a) | (nb >= b)]

    lo, hi = bounds[rank]
    mine = needs_of(rank)
    halo = {int(p): mine[owner[mine] == p] for p in np.unique(owner[mine])}
    send = {}
    for p in range(world):
        if p == rank:
            continue
        theirs = needs_of(p)
        rows = theirs[(theirs >= lo) & (theirs < hi)]
        if rows.size:
            send[p] = rows
    return NodePartition(world, rank, lo, hi, owner, halo, send)


def exchange_rows(part: NodePartition, buf, stage_slice=None, group=None):
    """Fill the halo rows of ``buf`` (node-major tensor, first dim = node) from
    their owners with one grouped batch of point-to-point ops.
    ``stage_slice`` optionally selects a sub-block of each node row (e.g. one
    horizon stage of the Gamma work array)."""
    import torch
    import torch.distributed as dist

    def rows(ids):
        idx = torch.as_tensor(ids, device=buf.device)
        v = buf.index_select(0, idx)
        return v if stage_slice is None else v[:, stage_slice]

    ops, recvs = [], []
    for p, ids in sorted(part.send.items()):
        ops.append(dist.P2POp(dist.isend, rows(ids).contiguous(), p, group))
    for p, ids in sorted(part.halo.items()):
        tmpl = rows(ids)
        r = torch.empty_like(tmpl.contiguous())
        ops.append(dist.P2POp(dist.irecv, r, p, group))
        recvs.append((ids, r))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for ids, r in recvs:
        idx = torch.as_tensor(ids, device=buf.device)
        if stage_slice is None:
            buf.index_copy_(0, idx, r)
        else:
            view = buf[:, stage_slice]
            view.index_copy_(0, idx, r)


def allreduce_sum(t, group=None):
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_owned(part: NodePartition, buf, group=None):
    """Replicate a node-major tensor whose rows [lo, hi) are valid on each rank."""
    import torch
    import torch.distributed as dist

    M = buf.shape[0]
    bounds = [shard_range(M, part.world, r) for r in range(part.world)]
    rows = max(b - a for a, b in bounds)  # all_gather needs equal sizes: pad
    a0, b0 = bounds[part.rank]
    mine = torch.zeros((rows,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
    mine[: b0 - a0].copy_(buf[a0:b0])
    out = [torch.empty_like(mine) for _ in bounds]
    dist.all_gather(out, mine, group=group)
    for (a, b), c in zip(bounds, out):
        buf[a:b].copy_(c[: b - a])
    return buf


class PartitionedCondenser:
    """GPU node-partitioned recursion + cost for one rank (NCCL).

    Wraps the single-device kernels with a node range (gm_set_node_range)
    and the exchanges above.  ``run(lin_blocks, x0, spec_dev)`` returns the
    all-reduced (H0, g0) and the work array whose owned + halo rows are valid."""

    def __init__(self, eng, part: NodePartition, N: int, nx: int, nu: int):
        from ._runtime import lib

        self.eng, self.part, self.N, self.nx, self.nu = eng, part, N, nx, nu
        self.ld = lib().gm_gamma_ld(N, nu)
        eng.ctx.call("gm_set_node_range", part.lo, part.hi)
        self.W = eng.zeros((eng.M, N + 1, nx, self.ld), np.float32)

    def gammas(self, a_self, a_nbr, b, c, x0):
        eng, N = self.eng, self.N
        sp = eng.stream_ptr()
        for n in range(-1, N):
            eng.ctx.call("gm_condense_gammas_stage", 1, N, n, a_self.data_ptr(),
                         a_nbr.data_ptr() if eng.E else None, b.data_ptr(), c.data_ptr(),
                         x0.data_ptr(), self.W.data_ptr(), self.ld, sp)
            # stage n+1 rows of the halo are needed by stage n+2
            exchange_rows(self.part, self.W, stage_slice=n + 1)
        return self.W

    def cost(self, ds, H0, g0):
        eng, N = self.eng, self.N
        partial = 0 if self.part.rank == 0 else 1
        eng.ctx.call("gm_condense_cost", 1, N, self.W.data_ptr(), self.ld, ds.q.data_ptr(), 0,
                     ds.x_ref.data_ptr(), 0, ds.r.data_ptr(), 0, ds.u_ref.data_ptr(), 0,
                     H0.data_ptr(), g0.data_ptr(), partial, eng.stream_ptr())
        allreduce_sum(H0)
        allreduce_sum(g0)
        return H0, g0


class PartitionedMpc:
    """One RTI step (mpc.py:102-200) of a node-partitioned instance, one rank
    per GPU.  The linearisation trajectory, the QP and the applied input are
    replicated; per-node work (K-LIN, K-REC, K-HG, state-constraint rows) is
    done for owned nodes only, with the exchanges described in the module
    docstring.  Requires an initialised torch.distributed process group
    (world size 1 works and degenerates to the single-device path)."""

    def __init__(self, model, topo, spec, cfg, part: NodePartition, device=None):
        import ctypes

        from . import device as _dev
        from .condensing import device_spec

        self.eng = eng = _dev.engine(topo, model, device)
        self.model, self.topo, self.spec, self.cfg, self.part = model, topo, spec, cfg, part
        N, nx, nu = cfg.horizon, 2 * model.n_p, model.n_u
        self.N, self.nx, self.nu = N, nx, nu
        eng.set_dims(nx, nu)
        self.cond = PartitionedCondenser(eng, part, N, nx, nu)
        self.ds = ds = device_spec(eng, spec, nx, nu)
        rows = ds.rows
        M, E = eng.M, eng.E
        f32, f64, i32 = np.float32, np.float64, np.int32
        e = eng.empty
        self.n0, self.m0, self.ns = N * nu, rows.m0, ds.ns
        self.n, self.m = self.n0 + self.ns, self.m0 + self.ns
        self.ls = e((N + 1, M, nx), f64)
        self.li = e((N, nu), f64)
        self.x0 = e((M, nx), f64)
        self.a_self = e((N, M, nx, nx), f32)
        self.a_nbr = e((N, max(E, 1), nx, nx), f32)
        self.b = e((N, M, nx, nu), f32)
        self.c = e((N, M, nx), f64)
        self.H0 = e((self.n0, self.n0), f64)
        self.g0 = e((self.n0,), f64)
        self.C0 = e((max(self.m0, 1), self.n0), f64)
        self.d0 = e((max(self.m0, 1),), f64)
        # row ownership: input rows by rank 0, state rows by the owner of their node
        own = np.zeros(max(self.m0, 1))
        own[: rows.n_in] = 1.0 if part.rank == 0 else 0.0
        if rows.n_st:
            own[rows.n_in: self.m0] = (part.owner[rows.st_node] == part.rank).astype(float)
        self.row_mask = eng.h2d(own, f64)
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
        self.planned_states = e((M, N + 1, nx), f64)
        self.planned_inputs = e((N, nu), f64)
        self.next_states = e((N + 1, M, nx), f64)
        self.next_inputs = e((N, nu), f64)
        self.u_applied = e((nu,), f64)
        self.u_prev = eng.zeros((nu,), f64)
        self.summary = e((nu + 2,), f64)
        self.settings_c = cfg.solver.as_c()
        self._ctypes = ctypes

    def step(self, x_measured, lin_states, lin_inputs):
        """x_measured (M, nx); lin_states (N+1, M, nx); lin_inputs (N, nu)
        (numpy or device tensors, replicated on every rank).  Returns
        (u_applied, status_code, iterations); the successor trajectory is in
        ``next_states`` / ``next_inputs`` (replicated)."""
        import torch

        from .condensing import cost_device, rows_device  # noqa: F401

        eng, N, nu, ds = self.eng, self.N, self.nu, self.ds
        ctx, sp = eng.ctx, eng.stream_ptr()
        for dst, src in ((self.x0, x_measured), (self.ls, lin_states), (self.li, lin_inputs)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
                      if isinstance(src, np.ndarray) else src)
        self.ls[0].copy_(self.x0)
        ctx.call("gm_set_node_range", self.part.lo, self.part.hi)
        ctx.call("gm_linearize", N, self.ls.data_ptr(), self.li.data_ptr(), self.a_self.data_ptr(),
                 self.a_nbr.data_ptr() if eng.E else None, self.b.data_ptr(), self.c.data_ptr(),
                 None, sp)
        if self.part.world == 1:
            # nothing to exchange: the fused persistent recursion + cost kernel
            # (K-COND) replaces the per-stage launches and the Gamma re-read
            from .condensing import fused_device

            W = self.cond.W
            fused_device(eng, ds, self.a_self, self.a_nbr if eng.E else None, self.b, self.c,
                         self.x0, W, self.cond.ld, N, self.H0, self.g0)
        else:
            W = self.cond.gammas(self.a_self, self.a_nbr, self.b, self.c, self.x0)
            self.cond.cost(ds, self.H0, self.g0)
        if self.m0:
            rows_device(eng, ds, W, self.cond.ld, N, self.C0, self.d0)
            self.C0.mul_(self.row_mask[:, None])
            self.d0.mul_(self.row_mask)
            allreduce_sum(self.C0)
            allreduce_sum(self.d0)
        if self.ns:
            ctx.call("gm_expand_soft", 1, self.n0, self.m0, self.H0.data_ptr(), self.g0.data_ptr(),
                     self.C0.data_ptr(), self.d0.data_ptr(), self.ns, ds.idx.data_ptr(),
                     ds.rho1.data_ptr(), ds.rho2.data_ptr(), self.H.data_ptr(), self.g.data_ptr(),
                     self.C.data_ptr(), self.d.data_ptr(), sp)
        warm = None
        if self.cfg.warm_start:
            self.warm[: N * nu].copy_(self.li.reshape(-1))
            warm = self.warm.data_ptr()
        ctx.call("gm_solve_qp", 1, self.n, self.m, self.H.data_ptr(), self.g.data_ptr(),
                 self.C.data_ptr() if self.m else None, self.d.data_ptr() if self.m else None, warm,
                 self._ctypes.byref(self.settings_c), self.u.data_ptr(), self.lam.data_ptr(),
                 self.status.data_ptr(), self.iters.data_ptr(), self.resid.data_ptr(), sp)
        ctx.call("gm_mpc_finish", 1, N, W.data_ptr(), self.cond.ld, self.u.data_ptr(), self.n,
                 self.status.data_ptr(), self.iters.data_ptr(), self.ls.data_ptr(),
                 self.li.data_ptr(), self.ls.data_ptr(), self.li.data_ptr(),
                 float(self.cfg.sqp_damping),
                 0 if self.cfg.fallback == "hold-previous-input" else 1, self.u_prev.data_ptr(), 1,
                 None, self.planned_states.data_ptr(), self.planned_inputs.data_ptr(),
                 self.next_states.data_ptr(), self.next_inputs.data_ptr(),
                 self.u_applied.data_ptr(), self.summary.data_ptr(), sp)
        if self.part.world > 1:
            # owned node rows of the plan are valid here: replicate, then shift
            # (at world size 1 gm_mpc_finish already wrote the whole shift)
            gather_owned(self.part, self.planned_states)
            ps = self.planned_states.transpose(0, 1)  # (N+1, M, nx)
            self.next_states[:N].copy_(ps[1:])
            self.next_states[N].copy_(ps[N])
        ctx.call("gm_set_node_range", 0, eng.M)
        summ = self.summary.cpu().numpy()
        return summ[:nu].copy(), int(summ[nu]), int(summ[nu + 1])
