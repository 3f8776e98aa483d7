"""Batched training gradients of the dynamics model on the GPU.

Mirrors ``gnnmpc/training.py``: ``_weight_grid`` (``:56-67``), ``params_of``
(= ``_params``, ``:95-96``) and ``loss_gradients`` (``:99-150``) -- the batch
loss ``sum(W r^2)/B + lambda |p|^2`` of the one-step prediction and its
gradient with respect to every parameter, reverse mode through the
message-passing step, computed by the library's K-TRAIN kernels
(``csrc/k_train.cu``, fp64 like the reference).  The Adam loop, datasets
and early stopping (``:153-280``) are offline host logic outside the
per-step hot path and are not mirrored.
"""

from __future__ import annotations

import numpy as np

from . import device as _dev
from ._runtime import lib


def _weight_grid(config_weights, node_count: int, n_state: int) -> np.ndarray:
    """Diagonal of O expanded to an (M, n_state) grid (``training.py:56-67``)."""
    if config_weights is None:
        return np.ones((node_count, n_state))
    w = np.atleast_1d(np.asarray(config_weights, dtype=float))
    if w.size == 1:
        return np.full((node_count, n_state), w[0])
    if w.size == n_state:
        return np.tile(w, (node_count, 1))
    if w.size == node_count * n_state:
        return w.reshape(node_count, n_state)
    raise ValueError("state weights must be scalar, per-feature or per-component")


def params_of(model) -> list:
    """Parameter list in gradient order (``training.py:95-96``)."""
    return model.psi.weights + model.psi.biases + model.phi.weights + model.phi.biases


def loss_gradients(model, topo, X, U, Xn, weights, l2_lambda: float):
    """Batch loss and its gradient w.r.t. every parameter, in the order of
    ``params_of`` (``training.py:99-150``).  X, Xn (B, M, n_state), U (B, n_u),
    weights (M, n_state)."""
    X = np.asarray(X, dtype=float)
    if X.ndim != 3 or X.shape[0] == 0:
        raise ValueError("X must be a non-empty (B, M, n_state) batch")
    if l2_lambda < 0:
        raise ValueError("l2_lambda must be nonnegative")
    eng = _dev.engine(topo, model)
    B = X.shape[0]
    P = int(lib().gm_param_count(eng.ctx.handle))
    f64 = np.float64
    dX, dU, dXn = eng.h2d(X, f64), eng.h2d(np.asarray(U, dtype=float).reshape(B, -1), f64), \
        eng.h2d(np.asarray(Xn, dtype=float).reshape(X.shape), f64)
    dW = eng.h2d(np.asarray(weights, dtype=float).reshape(X.shape[1:]), f64)
    loss = eng.empty((1,), f64)
    grads = eng.empty((P,), f64)
    eng.ctx.call("gm_loss_gradients", B, dX.data_ptr(), dU.data_ptr(), dXn.data_ptr(),
                 dW.data_ptr(), float(l2_lambda), loss.data_ptr(), grads.data_ptr(),
                 eng.stream_ptr())
    flat = grads.cpu().numpy()
    out, o = [], 0
    for p in params_of(model):
        n = int(np.size(p))
        out.append(flat[o:o + n].reshape(np.shape(p)))
        o += n
    return float(loss.cpu().numpy()[0]), out
