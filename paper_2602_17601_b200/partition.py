"""Node-partitioned RTI step for graphs too large for one device (cfg5).

The horizon recursion is sequential in the stage index but node-parallel
within a stage (condensing.py:211-224): node i at stage n+1 reads
only the stage-n rows of its closed neighbourhood.  The reference splits the
nodes of one stage over a thread pool in contiguous chunks
(condensing.py:208-227); here the chunks are contiguous id ranges (row slabs of
the 2-D mesh) owned by one GPU each.

Each rank works on its *local graph*: its owned nodes [lo, hi) plus its halo
(the in-neighbours of owned nodes owned elsewhere), renumbered in ascending
global id order -- halo below, owned, halo above -- so the owned nodes are the
contiguous local range [own_lo, own_hi) and every per-node array holds
owned + halo rows only (no full-M buffers).  Halo nodes have no in-edges in
the local graph; their rows arrive from their owners.

Per RTI step, on every rank:

1. K-LIN over the owned nodes (halo states are local: the trajectory of
   owned + halo nodes is kept on the rank);
2. stage 0 of the Gamma work array for all local nodes (it is x0), then per
   stage n+1: K-REC over the owned nodes, pack the boundary rows other ranks
   read (our gather kernel, device index lists built once), one grouped
   point-to-point exchange, unpack into the halo rows (scatter kernel);
3. K-HG partial over the owned nodes (rank 0 adds R-bar / r_lin), K-CON with
   the rows of non-owned nodes masked, then ONE all-reduce(sum) of
   [H | g | C | d];
4. the small QP solved redundantly on every rank (identical inputs and a
   deterministic kernel give identical outputs: no broadcast);
5. K-RS over all local nodes: the halo's Gamma rows are already exchanged for
   every stage, so the planned / shifted trajectory of owned AND halo nodes
   is formed locally -- no trajectory all-gather between steps.

The data plane goes through a transport object: ``DistTransport``
(torch.distributed: NCCL over NVLink between GPUs, gloo on CPU) or
``LocalTransport`` (ranks as threads of one process sharing one device, for
tests: device-to-device copies behind a barrier, no kernel ever waits on
another rank's kernel).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from .batch import shard_range
from . import device as _dev
from .device import topology_csr
from .errors import ConfigurationError


# ---------------------------------------------------------------------------
# partition plan
# ---------------------------------------------------------------------------

@dataclass
class NodePartition:
    world: int
    rank: int
    lo: int
    hi: int
    owner: np.ndarray          # (M,) rank owning each node
    halo: dict                 # peer rank -> global node ids this rank receives (ascending)
    send: dict                 # peer rank -> global node ids this rank sends (ascending)
    local_nodes: np.ndarray = None   # global ids of the local nodes (ascending)
    node_map: np.ndarray = None      # global id -> local id (-1: not local)
    own_lo: int = 0                  # owned nodes = local [own_lo, own_hi)
    own_hi: int = 0
    _local_topo: object = field(default=None, repr=False)

    @property
    def owned(self) -> np.ndarray:
        return np.arange(self.lo, self.hi)

    @property
    def node_count(self) -> int:
        return int(self.owner.shape[0])

    def local_topology(self, topo):
        """The rank's local graph: owned nodes keep their in-neighbour lists
        (mapped to local ids, order preserved since the map is monotone),
        halo nodes have none.  Cached on the partition."""
        if self._local_topo is None:
            from .graph import GraphTopology

            nm = self.node_map
            nbrs = []
            for g in self.local_nodes:
                if self.lo <= g < self.hi:
                    nbrs.append(tuple(int(nm[j]) for j in topo.in_neighbors[g]))
                else:
                    nbrs.append(())
            self._local_topo = GraphTopology(len(nbrs), tuple(nbrs), int(topo.neighbor_bound))
        return self._local_topo

    def local_rows(self, arr, axis=0):
        """Rows of a global per-node array that belong to this rank's local
        graph (numpy or torch)."""
        if hasattr(arr, "index_select") and not isinstance(arr, np.ndarray):
            import torch

            idx = torch.as_tensor(self.local_nodes, device=arr.device)
            return arr.index_select(axis, idx)
        return np.take(np.asarray(arr), self.local_nodes, axis=axis)


def partition_nodes(topo, world: int, rank: int) -> NodePartition:
    """Contiguous id ranges; halo = in-neighbours of owned nodes owned elsewhere."""
    M = topo.node_count
    if not 0 <= rank < world:
        raise ConfigurationError("rank out of range")
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
    local = np.concatenate([mine[mine < lo], np.arange(lo, hi), mine[mine >= hi]]).astype(np.int64)
    node_map = np.full(M, -1, dtype=np.int64)
    node_map[local] = np.arange(local.size)
    own_lo = int(np.sum(mine < lo))
    return NodePartition(world, rank, lo, hi, owner, halo, send, local, node_map, own_lo,
                         own_lo + (hi - lo))


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class DistTransport:
    """torch.distributed data plane (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def sendrecv(self, sends: dict, recvs: dict):
        """One grouped batch of point-to-point ops: sends[peer] -> peer,
        recvs[peer] <- peer."""
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, p, self.group) for p, t in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, t, p, self.group) for p, t in sorted(recvs.items())]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, outs: list, t):
        self.dist.all_gather(outs, t, group=self.group)


class NcclTransport:
    """Native data plane (``gm_init_comm`` / ``gm_sendrecv`` /
    ``gm_allreduce_sum``): an NCCL communicator in its own native context on
    this rank's device, every operation enqueued on the caller's current
    stream with no host synchronisation -- so a rank's whole step (kernels and
    exchanges) can be captured in one CUDA graph, which ``DistTransport``'s
    waits do not allow.  The 128-byte NCCL id comes from ``unique_id`` or is
    broadcast from rank 0 over an initialised torch.distributed group."""

    def __init__(self, rank: int, world: int, device=None, unique_id: bytes | None = None, group=None):
        import ctypes

        import torch

        from ._runtime import Context, lib

        self.torch, self.rank, self.world = torch, int(rank), int(world)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device.index if hasattr(device, "index") else int(device)))
        if not lib().gm_comm_available():
            raise RuntimeError("libnccl.so.2 not found: the native data plane needs NCCL")
        if unique_id is None:
            import torch.distributed as dist

            buf = (ctypes.c_uint8 * 128)()
            if self.rank == 0 and lib().gm_comm_unique_id(ctypes.addressof(buf)) != 0:
                raise RuntimeError("ncclGetUniqueId failed")
            t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device=self.device)
            dist.broadcast(t, 0, group=group)
            unique_id = bytes(t.cpu().tolist())
        if len(unique_id) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        self._id = (ctypes.c_uint8 * 128)(*unique_id)
        self.ctx = Context(self.device.index)
        self.ctx.call("gm_init_comm", ctypes.addressof(self._id), self.rank, self.world)
        self._ct = ctypes

    @staticmethod
    def unique_id() -> bytes:
        """A fresh NCCL id (rank 0), to hand to the other ranks out of band."""
        import ctypes

        from ._runtime import lib

        buf = (ctypes.c_uint8 * 128)()
        if lib().gm_comm_unique_id(ctypes.addressof(buf)) != 0:
            raise RuntimeError("ncclGetUniqueId failed (is libnccl.so.2 present?)")
        return bytes(buf)

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def sendrecv(self, sends: dict, recvs: dict):
        """One grouped batch: sends[peer] -> peer, recvs[peer] <- peer
        (contiguous device tensors, sizes in bytes from the tensors)."""
        ct = self._ct
        sp = sorted(sends.items())
        rp = sorted(recvs.items())

        def arrays(items):
            n = len(items)
            peers = (ct.c_int * max(n, 1))(*[p for p, _ in items])
            bufs = (ct.c_void_p * max(n, 1))(*[t.data_ptr() for _, t in items])
            nbytes = (ct.c_int64 * max(n, 1))(*[t.numel() * t.element_size() for _, t in items])
            return n, peers, bufs, nbytes

        ns, sp_, sb, sn = arrays(sp)
        nr, rp_, rb, rn = arrays(rp)
        self.ctx.call("gm_sendrecv", ns, ct.addressof(sp_), ct.addressof(sb), ct.addressof(sn), nr,
                      ct.addressof(rp_), ct.addressof(rb), ct.addressof(rn), self._stream())

    def allreduce_sum(self, t):
        if t.dtype != self.torch.float64 or not t.is_contiguous():
            raise ValueError("allreduce_sum: contiguous float64 tensors only")
        self.ctx.call("gm_allreduce_sum", t.data_ptr(), t.numel(), self._stream())
        return t

    def all_gather(self, outs: list, t):
        """outs[r] <- rank r's t: one grouped batch of sends to / receives
        from every rank (own slot by copy)."""
        outs[self.rank].copy_(t)
        peers = [r for r in range(self.world) if r != self.rank]
        self.sendrecv({p: t for p in peers}, {p: outs[p] for p in peers})

    def close(self):
        if self.ctx is not None:
            self.ctx.call("gm_comm_destroy")
            self.ctx.close()
            self.ctx = None


class LocalHub:
    """Shared state of the in-process ranks of a LocalTransport group."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class LocalTransport:
    """Ranks as threads of one process (one device or CPU): every collective
    is a barrier, device-to-device copies from the peers' posted tensors and
    a second barrier.  Each rank synchronises its own stream before posting,
    so no kernel ever waits on another rank's kernel.  Sums are taken in
    rank order (deterministic)."""

    def __init__(self, hub: LocalHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    @staticmethod
    def _sync(t):
        if t is not None and getattr(t, "is_cuda", False):
            import torch

            torch.cuda.current_stream(t.device).synchronize()

    def _post(self, obj, probe):
        self._sync(probe)
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()

    def _done(self, probe):
        self._sync(probe)
        self.hub.barrier.wait()

    def sendrecv(self, sends: dict, recvs: dict):
        probe = next(iter(sends.values()), None)
        if probe is None:
            probe = next(iter(recvs.values()), None)
        self._post(sends, probe)
        for p, buf in recvs.items():
            buf.copy_(self.hub.slots[p][self.rank])
        self._done(probe)

    def allreduce_sum(self, t):
        self._post(t, t)
        acc = self.hub.slots[0].clone()
        for r in range(1, self.world):
            acc += self.hub.slots[r]
        self._done(t)
        t.copy_(acc)
        self._sync(t)
        return t

    def all_gather(self, outs: list, t):
        self._post(t, t)
        for r in range(self.world):
            outs[r].copy_(self.hub.slots[r])
        self._done(t)


# ---------------------------------------------------------------------------
# halo exchange of node-major rows
# ---------------------------------------------------------------------------

class HaloExchange:
    """Per-peer index lists (local ids) and pack / unpack buffers for the
    rows of one horizon stage of a node-major array ``buf`` (first dim =
    local node).  On CUDA tensors the pack / unpack run in the library's
    gather / scatter kernels (``gm_gather_rows`` / ``gm_scatter_rows``)
    with the index lists resident on the device; ``torch_pack=True`` uses
    torch indexing instead (CPU tensors: the gloo host-logic tests)."""

    def __init__(self, part: NodePartition, buf, transport, eng=None, torch_pack=False):
        import torch

        self.part, self.buf, self.tr, self.eng = part, buf, transport, eng
        self.torch_pack = torch_pack or not buf.is_cuda
        dev = buf.device
        nm = part.node_map
        self.send_idx = {p: torch.as_tensor(nm[ids].astype(np.int32), device=dev)
                         for p, ids in part.send.items()}
        self.recv_idx = {p: torch.as_tensor(nm[ids].astype(np.int32), device=dev)
                         for p, ids in part.halo.items()}
        row_shape = tuple(buf.shape[2:])
        self.sbuf = {p: torch.empty((len(i),) + row_shape, dtype=buf.dtype, device=dev)
                     for p, i in self.send_idx.items()}
        self.rbuf = {p: torch.empty((len(i),) + row_shape, dtype=buf.dtype, device=dev)
                     for p, i in self.recv_idx.items()}
        es = buf.element_size()
        self.row_bytes = int(np.prod(row_shape)) * es if row_shape else es
        self.node_stride = buf.stride(0) * es
        self.stage_stride = buf.stride(1) * es

    def exchange(self, stage: int):
        """Halo rows of ``buf[:, stage]`` from their owners."""
        b = self.buf
        if self.torch_pack:
            for p, idx in self.send_idx.items():
                self.sbuf[p].copy_(b[:, stage].index_select(0, idx.long()))
        else:
            ctx, sp = self.eng.ctx, self.eng.stream_ptr()
            base = b.data_ptr() + stage * self.stage_stride
            for p, idx in self.send_idx.items():
                ctx.call("gm_gather_rows", base, self.sbuf[p].data_ptr(), idx.data_ptr(), idx.numel(),
                         self.row_bytes, self.node_stride, 1, 0, sp)
        self.tr.sendrecv(self.sbuf, self.rbuf)
        if self.torch_pack:
            view = b[:, stage]
            for p, idx in self.recv_idx.items():
                view.index_copy_(0, idx.long(), self.rbuf[p])
        else:
            ctx, sp = self.eng.ctx, self.eng.stream_ptr()
            base = b.data_ptr() + stage * self.stage_stride
            for p, idx in self.recv_idx.items():
                ctx.call("gm_scatter_rows", self.rbuf[p].data_ptr(), base, idx.data_ptr(), idx.numel(),
                         self.row_bytes, self.node_stride, 1, 0, sp)


# ---------------------------------------------------------------------------
# the partitioned RTI step
# ---------------------------------------------------------------------------

class PartitionedMpc:
    """One RTI step (mpc.py:102-200) of a node-partitioned instance, one rank
    per GPU (or per thread with a LocalTransport).  The QP and the applied
    input are replicated; per-node work is done for owned nodes, with the
    exchanges described in the module docstring.  ``transport`` defaults to
    torch.distributed (an initialised process group); world size 1 runs the
    single-device fused condensing kernel."""

    def __init__(self, model, topo, spec, cfg, part: NodePartition, device=None, transport=None):
        import ctypes

        from . import device as _dev
        from ._runtime import lib
        from .condensing import DeviceSpec, spec_rows
        from .qpsolver import settings_c

        if cfg.sqp_iterations != 1 or cfg.input_filter_tau is not None:
            raise ConfigurationError("PartitionedMpc runs the RTI step: sqp_iterations == 1, "
                                     "no input filter")
        if part.world > 1 and transport is None:
            transport = DistTransport()
        self.transport = transport
        self.model, self.topo, self.spec, self.cfg, self.part = model, topo, spec, cfg, part
        self.ltopo = ltopo = part.local_topology(topo) if part.world > 1 else topo
        # a private engine (context) per rank: the node range below is context
        # state and must not leak into other users of a cached engine
        self.eng = eng = _dev.Engine(ltopo, _dev.device_index(device))
        eng.bind_model(model)
        N, nx, nu = cfg.horizon, 2 * model.n_p, model.n_u
        self.N, self.nx, self.nu = N, nx, nu
        eng.set_dims(nx, nu)
        self.ld = lib().gm_gamma_ld(N, nu)
        ML, EL = eng.M, eng.E
        self.ML = ML
        self.own = (part.own_lo, part.own_hi) if part.world > 1 else (0, ML)
        grow = spec_rows(spec, nx, nu)
        if part.world > 1:
            self.ds = ds = DeviceSpec(eng, spec, nx, nu, part.local_nodes, part.node_map)
        else:
            self.ds = ds = DeviceSpec(eng, spec, nx, nu)
        rows = ds.rows
        f32, f64, i32 = np.float32, np.float64, np.int32
        e = eng.empty
        self.n0, self.m0, self.ns = N * nu, rows.m0, ds.ns
        self.n, self.m = self.n0 + self.ns, self.m0 + self.ns
        self.ls = e((N + 1, ML, nx), f64)
        self.li = e((N, nu), f64)
        self.x0 = e((ML, nx), f64)
        self.a_self = e((N, ML, nx, nx), f32)
        self.a_nbr = e((N, max(EL, 1), nx, nx), f32)
        self.b = e((N, ML, nx, nu), f32)
        self.c = e((N, ML, nx), f64)
        self.W = eng.zeros((ML, N + 1, nx, self.ld), f32)
        # [H0 | g0 | C0 | d0] in one buffer: one all-reduce per step
        n0, m0 = self.n0, max(self.m0, 1)
        self.red = e((n0 * n0 + n0 + m0 * n0 + m0,), f64)
        o = 0
        self.H0 = self.red[o:o + n0 * n0].view(n0, n0); o += n0 * n0
        self.g0 = self.red[o:o + n0]; o += n0
        self.C0 = self.red[o:o + m0 * n0].view(m0, n0); o += m0 * n0
        self.d0 = self.red[o:o + m0]
        # row ownership: input rows by rank 0, state rows by the owner of their node
        own = np.zeros(m0)
        own[: grow.n_in] = 1.0 if part.rank == 0 else 0.0
        if grow.n_st:
            own[grow.n_in: self.m0] = (part.owner[grow.st_node] == part.rank).astype(float)
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
        self.planned_states = e((ML, N + 1, nx), f64)
        self.planned_inputs = e((N, nu), f64)
        self.next_states = e((N + 1, ML, nx), f64)
        self.next_inputs = e((N, nu), f64)
        self.u_applied = e((nu,), f64)
        self.u_prev = eng.zeros((nu,), f64)
        self.has_prev = 0
        self.summary = e((nu + 2,), f64)
        self.settings_c = settings_c(cfg.solver)
        self._ctypes = ctypes
        self.halo = HaloExchange(part, self.W, transport, eng) if part.world > 1 else None
        self._graphs = {}

    # -- inputs ----------------------------------------------------------------
    def _local(self, arr, axis):
        """Accept global (M rows) or local (owned + halo rows) per-node arrays."""
        if self.part.world > 1 and arr.shape[axis] == self.part.node_count \
                and arr.shape[axis] != self.ML:
            return self.part.local_rows(arr, axis)
        return arr

    def load(self, x_measured, lin_states, lin_inputs, last_applied=None):
        import torch

        for dst, src, ax in ((self.x0, x_measured, 0), (self.ls, lin_states, 1),
                             (self.li, lin_inputs, None)):
            if ax is not None:
                src = self._local(src, ax)
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
                      if isinstance(src, np.ndarray) else src)
        self.ls[0].copy_(self.x0)
        self.has_prev = 0 if last_applied is None else 1
        if last_applied is not None:
            self.u_prev.copy_(torch.as_tensor(np.asarray(last_applied, dtype=np.float64)
                                              if isinstance(last_applied, np.ndarray) else last_applied))

    # -- the step --------------------------------------------------------------
    def step(self, x_measured, lin_states, lin_inputs, last_applied=None):
        """x_measured (M|ML, nx); lin_states (N+1, M|ML, nx); lin_inputs (N, nu)
        (numpy or device tensors; global arrays are sliced to the local
        nodes).  Returns (u_applied, status_code, iterations); the successor
        trajectory of the local nodes is in ``next_states`` / ``next_inputs``
        (pass them back as the next step's lin_states / lin_inputs)."""
        self.load(x_measured, lin_states, lin_inputs, last_applied)
        self.enqueue()
        summ = self.summary.cpu().numpy()
        nu = self.nu
        return summ[:nu].copy(), int(summ[nu]), int(summ[nu + 1])

    def capture(self):
        """Record ``enqueue`` as one CUDA graph -- K-LIN, the per-stage K-REC
        launches with their halo pack / NCCL exchange / unpack, K-HG, the
        all-reduce, K-QP and K-RS -- for the current ``has_prev``.  Needs a
        stream-ordered data plane: ``NcclTransport`` (or world 1)."""
        import torch

        if self.part.world > 1 and not isinstance(self.transport, NcclTransport):
            raise ConfigurationError("CUDA-graph capture of the partitioned step needs NcclTransport")
        self.enqueue()  # first launches (lazy allocations) outside the capture
        torch.cuda.current_stream(self.eng.device).synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.enqueue()
        self._graphs[self.has_prev] = g
        return g

    def step_graph(self, x_measured, lin_states, lin_inputs, last_applied=None):
        """``step`` through the captured graph (captured on first use)."""
        self.load(x_measured, lin_states, lin_inputs, last_applied)
        g = self._graphs.get(self.has_prev) or self.capture()
        g.replay()
        summ = self.summary.cpu().numpy()
        nu = self.nu
        return summ[:nu].copy(), int(summ[nu]), int(summ[nu + 1])

    def enqueue(self, events=None):
        """The whole step on the current stream; host synchronisation only
        inside the transport's collectives.  ``events`` (5 torch.cuda.Event,
        optional) bracket K-LIN | condensing incl. exchanges and all-reduce |
        K-QP | K-RS."""
        from .condensing import fused_device, rows_device

        eng, N, nu, ds = self.eng, self.N, self.nu, self.ds
        ctx, sp = eng.ctx, eng.stream_ptr()
        lo, hi = self.own
        a_nbr = self.a_nbr.data_ptr() if eng.E else None

        def mark(i):
            if events is not None:
                events[i].record()

        try:
            ctx.call("gm_set_node_range", lo, hi)
            mark(0)
            ctx.call("gm_linearize", N, self.ls.data_ptr(), self.li.data_ptr(),
                     self.a_self.data_ptr(), a_nbr, self.b.data_ptr(), self.c.data_ptr(), None, sp)
            mark(1)
            if self.part.world == 1:
                # nothing to exchange: the fused persistent recursion + cost
                # kernel (K-COND) replaces the per-stage launches
                ctx.call("gm_set_node_range", 0, self.ML)
                fused_device(eng, ds, self.a_self, self.a_nbr if eng.E else None, self.b, self.c,
                             self.x0, self.W, self.ld, N, self.H0, self.g0)
            else:
                # stage 0 (x0) for every local node, halo included
                ctx.call("gm_set_node_range", 0, self.ML)
                self._stage(-1)
                ctx.call("gm_set_node_range", lo, hi)
                for n in range(N):
                    self._stage(n)
                    self.halo.exchange(n + 1)
                partial = 0 if self.part.rank == 0 else 1
                ctx.call("gm_condense_cost", 1, N, self.W.data_ptr(), self.ld, ds.q.data_ptr(), 0,
                         ds.x_ref.data_ptr(), 0, ds.r.data_ptr(), 0, ds.u_ref.data_ptr(), 0,
                         self.H0.data_ptr(), self.g0.data_ptr(), partial, sp)
            if self.m0:
                rows_device(eng, ds, self.W, self.ld, N, self.C0, self.d0)
            if self.part.world > 1:
                if self.m0:
                    self.C0.mul_(self.row_mask[:, None])
                    self.d0.mul_(self.row_mask)
                self.transport.allreduce_sum(self.red)
        finally:
            ctx.call("gm_set_node_range", 0, self.ML)
        if self.ns:
            ctx.call("gm_expand_soft", 1, self.n0, self.m0, self.H0.data_ptr(), self.g0.data_ptr(),
                     self.C0.data_ptr(), self.d0.data_ptr(), self.ns, ds.idx.data_ptr(),
                     ds.rho1.data_ptr(), ds.rho2.data_ptr(), self.H.data_ptr(), self.g.data_ptr(),
                     self.C.data_ptr(), self.d.data_ptr(), sp)
        mark(2)
        warm = None
        if self.cfg.warm_start:
            self.warm[: N * nu].copy_(self.li.reshape(-1))
            warm = self.warm.data_ptr()
        ctx.call("gm_solve_qp", 1, self.n, self.m, self.H.data_ptr(), self.g.data_ptr(),
                 self.C.data_ptr() if self.m else None, self.d.data_ptr() if self.m else None, warm,
                 self._ctypes.byref(self.settings_c), self.u.data_ptr(), self.lam.data_ptr(),
                 self.status.data_ptr(), self.iters.data_ptr(), self.resid.data_ptr(), sp)
        mark(3)
        # every local node's Gamma rows are valid (halo rows exchanged), so the
        # plan and its shift are formed for owned + halo nodes here
        tail = (self.status.data_ptr(), self.iters.data_ptr(), self.ls.data_ptr(),
                self.li.data_ptr(), self.ls.data_ptr(), self.li.data_ptr(),
                float(self.cfg.sqp_damping),
                0 if self.cfg.fallback == "hold-previous-input" else 1, self.u_prev.data_ptr(),
                self.has_prev, None, self.planned_states.data_ptr(),
                self.planned_inputs.data_ptr(), self.next_states.data_ptr(),
                self.next_inputs.data_ptr(), self.u_applied.data_ptr(), self.summary.data_ptr(), sp)
        if self.part.world == 1 and _dev.use_rollout(self.ML * (N + 1), self.nx, nu):
            # one rank owns the whole graph: K-RS by linear rollout
            ctx.call("gm_mpc_finish_rollout", 1, N, self.a_self.data_ptr(), a_nbr, self.b.data_ptr(),
                     self.c.data_ptr(), self.x0.data_ptr(), self.u.data_ptr(), self.n, *tail)
        else:
            ctx.call("gm_mpc_finish", 1, N, self.W.data_ptr(), self.ld, self.u.data_ptr(), self.n,
                     *tail)
        mark(4)

    def _stage(self, n):
        eng = self.eng
        eng.ctx.call("gm_condense_gammas_stage", 1, self.N, n, self.a_self.data_ptr(),
                     self.a_nbr.data_ptr() if eng.E else None, self.b.data_ptr(), self.c.data_ptr(),
                     self.x0.data_ptr(), self.W.data_ptr(), self.ld, eng.stream_ptr())

    # -- outputs ---------------------------------------------------------------
    def owned_slice(self):
        """Local index range of the owned nodes."""
        return slice(*self.own)
