"""Device engines: one native context per (CUDA device, topology).

An ``Engine`` owns a ``gm_ctx`` with the graph's CSR tables uploaded once
(the reference rebuilds its index tables per call under an ``lru_cache``,
``gnn.py:107``) and the model weights, re-uploaded only when the model's
parameters change (a cheap byte-for-byte fingerprint, so in-place edits of a
``GnnModel`` are honoured exactly like the reference, which reads the arrays
on every call).  Device memory and streams come from PyTorch; all compute is
in the native library.
"""

from __future__ import annotations

import threading
import weakref
from collections import OrderedDict

import numpy as np

from ._runtime import Context, require_cuda

_engines: "OrderedDict[tuple, Engine]" = OrderedDict()
_lock = threading.Lock()
_MAX_ENGINES = 8


def topology_csr(topo):
    """In-neighbour CSR (ptr, src) in canonical edge order for any
    GraphTopology-like object (``graph.py:60-63``)."""
    if hasattr(topo, "csr"):
        return topo.csr()
    deg = np.fromiter((len(ns) for ns in topo.in_neighbors), dtype=np.int64,
                      count=topo.node_count)
    ptr = np.zeros(topo.node_count + 1, dtype=np.int64)
    np.cumsum(deg, out=ptr[1:])
    src = np.fromiter((j for ns in topo.in_neighbors for j in ns), dtype=np.int64,
                      count=int(ptr[-1]))
    return ptr, src


def _model_fingerprint(model) -> bytes:
    nrm = model.normalization
    parts = [np.array([model.dt, model.n_p, model.n_u, model.n_m], dtype=float)]
    for mlp in (model.psi, model.phi):
        parts.append(np.asarray(mlp.layer_dims, dtype=float))
        parts.extend(np.asarray(W, dtype=float).ravel() for W in mlp.weights)
        parts.extend(np.asarray(b, dtype=float).ravel() for b in mlp.biases)
    parts.extend(np.asarray(a, dtype=float).ravel() for a in
                 (nrm.state_mean, nrm.state_scale, nrm.input_mean, nrm.input_scale))
    return np.concatenate(parts).tobytes()


class Engine:
    def __init__(self, topo, device_index: int):
        torch = require_cuda()
        self.torch = torch
        self.device = torch.device("cuda", device_index)
        self.topo = topo  # keeps id(topo) alive for the cache key
        self.ctx = Context(device_index)
        ptr, src = topology_csr(topo)
        self.M = int(topo.node_count)
        self.E = int(ptr[-1])
        self.ctx.call("gm_set_graph", self.M, int(topo.neighbor_bound), ptr.ctypes.data,
                      src.ctypes.data if src.size else None)
        from ._runtime import lib
        self.dmax = int(lib().gm_max_degree(self.ctx.handle))
        self._model_fp = None
        self._frozen_ref = None
        self._dims = None
        self.lock = threading.RLock()
        self.cache = {}  # workspace / uploaded-constant cache (see mpc.py, condensing.py)

    # -- bindings -----------------------------------------------------------
    def bind_model(self, model):
        frozen = getattr(model, "_frozen", None)
        if frozen is not None and self._frozen_ref is not None and self._frozen_ref() is model \
                and frozen == (id(model.psi), id(model.phi), id(model.normalization), model.dt):
            return  # same frozen model object, nothing can have changed
        fp = _model_fingerprint(model)
        if fp == self._model_fp:
            self._frozen_ref = weakref.ref(model) if frozen is not None else None
            return
        nrm = model.normalization

        def flat(mlp):
            dims = np.asarray(mlp.layer_dims, dtype=np.int32)
            w = np.concatenate([np.ascontiguousarray(W, dtype=float).ravel() for W in mlp.weights])
            b = np.concatenate([np.ascontiguousarray(v, dtype=float).ravel() for v in mlp.biases])
            return dims, w, b

        pd, pw, pb = flat(model.psi)
        hd, hw, hb = flat(model.phi)
        stats = [np.ascontiguousarray(a, dtype=float) for a in
                 (nrm.state_mean, nrm.state_scale, nrm.input_mean, nrm.input_scale)]
        from ._runtime import lib

        gen = lib().gm_model_generation(self.ctx.handle)
        self._model_fp = None  # a failed upload leaves no valid binding
        self.ctx.call("gm_set_model", int(model.n_p), int(model.n_u), int(model.n_m), float(model.dt),
                      len(model.psi.weights), pd.ctypes.data, pw.ctypes.data, pb.ctypes.data,
                      len(model.phi.weights), hd.ctypes.data, hw.ctypes.data, hb.ctypes.data,
                      *[s.ctypes.data for s in stats])
        if lib().gm_model_generation(self.ctx.handle) != gen:
            # weight buffers moved (layer dims changed) or a scalar baked into
            # kernel arguments changed: every captured step graph is stale.
            # Same-shape parameter edits are copied in place by gm_set_model
            # and keep the graphs valid.
            self.drop_graphs()
        self._model_fp = fp
        self._frozen_ref = weakref.ref(model) if frozen is not None else None
        self._dims = (2 * int(model.n_p), int(model.n_u))

    def drop_graphs(self):
        """Forget every captured CUDA graph of this engine (StepPlans are
        re-captured on their next use)."""
        for key in [k for k in self.cache if isinstance(k, tuple) and k and k[0] == "plan"]:
            self.cache.pop(key, None)

    def set_dims(self, nx: int, nu: int):
        if self._dims != (nx, nu):
            self.ctx.call("gm_set_dims", int(nx), int(nu))
            self._dims = (nx, nu)

    # -- memory helpers -----------------------------------------------------
    def h2d(self, arr, dtype):
        a = np.ascontiguousarray(arr, dtype=dtype)
        if not a.flags.writeable:  # torch.from_numpy needs a writable buffer
            a = a.copy()
        return self.torch.from_numpy(a).to(self.device, non_blocking=False)

    def empty(self, shape, dtype):
        tdt = {np.float64: self.torch.float64, np.float32: self.torch.float32,
               np.int32: self.torch.int32}[dtype]
        return self.torch.empty(tuple(int(s) for s in shape), dtype=tdt, device=self.device)

    def zeros(self, shape, dtype):
        t = self.empty(shape, dtype)
        t.zero_()
        return t

    def stream_ptr(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream


_ROLLOUT_MIN = 1 << 20  # node-stages per launch from which K-RS rolls out instead of reading Gamma


def use_rollout(node_stages: int, nx: int, nu: int) -> bool:
    """K-RS by linear rollout (gm_mpc_finish_rollout) instead of Gamma rows
    (gm_mpc_finish): for large batches the stage blocks are ~5x fewer bytes
    than Gamma's rows (cfg4, cfg5).  GM_FIN_ROLLOUT=0/1 forces either."""
    import os

    env = os.environ.get("GM_FIN_ROLLOUT")
    if nx != 6 or nu != 6:
        return False
    if env is not None:
        return env == "1"
    return node_stages >= _ROLLOUT_MIN


def device_index(device=None) -> int:
    """CUDA device ordinal of ``device`` (None: the current device)."""
    torch = require_cuda()
    if device is None:
        return torch.cuda.current_device()
    idx = device.index if hasattr(device, "index") else device
    return torch.cuda.current_device() if idx is None else int(idx)


def engine(topo, model=None, device=None) -> Engine:
    """Cached engine for (device, topology); binds ``model`` if given."""
    dev = device_index(device)
    key = (dev, id(topo))
    with _lock:
        eng = _engines.get(key)
        if eng is None or eng.topo is not topo:
            eng = Engine(topo, dev)
            _engines[key] = eng
            while len(_engines) > _MAX_ENGINES:
                _engines.popitem(last=False)
        else:
            _engines.move_to_end(key)
    if model is not None:
        eng.bind_model(model)
    return eng
