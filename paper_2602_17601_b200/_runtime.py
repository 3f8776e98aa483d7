"""ctypes binding of ``libgnnmpc_b200.so`` (the C ABI in ``include/gnnmpc_b200.h``).

This is the only place the package touches the native library.  There is no
CPU fallback: if the library is missing, or no CUDA device is present, every
device entry point raises ``RuntimeError`` (loudly, by design).

Device memory, streams and host<->device copies are PyTorch's (plumbing);
every computation of the hot path runs in the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigurationError

_HERE = Path(__file__).resolve().parent
# GM_LIB_PATH: load another build of the same library (A/B measurements of
# kernel variants within one process environment); default the in-tree build
LIB_PATH = Path(os.environ["GM_LIB_PATH"]) if os.environ.get("GM_LIB_PATH") else _HERE / "lib" / "libgnnmpc_b200.so"

GM_OK, GM_ERR_CONFIG, GM_ERR_NUMERIC, GM_ERR_CUDA = 0, 2, 3, 4
QP_STATUS_NAMES = ("optimal", "max_iterations", "primal_infeasible", "numerical_failure")

_lib = None
_lib_lock = threading.Lock()

c_int, c_i64, c_double, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P = ctypes.c_void_p  # every array argument is passed as a raw address


class QpSettingsC(ctypes.Structure):
    _fields_ = [("tolerance", ctypes.c_double), ("max_iterations", ctypes.c_int32),
                ("regularization", ctypes.c_double), ("fraction_to_boundary", ctypes.c_double)]


# name -> (restype, argtypes); mirrors include/gnnmpc_b200.h
_SIGNATURES = {
    "gm_abi_version": (c_int, []),
    "gm_launch_count": (c_i64, []),
    "gm_event_times": (c_int, [c_int, P, P]),
    "gm_create": (c_int, [ctypes.POINTER(c_void_p), c_int]),
    "gm_destroy": (None, [c_void_p]),
    "gm_last_error": (ctypes.c_char_p, [c_void_p]),
    "gm_set_graph": (c_int, [c_void_p, c_i64, c_i64, P, P]),
    "gm_edge_count": (c_i64, [c_void_p]),
    "gm_max_degree": (c_i64, [c_void_p]),
    "gm_graph_tables": (c_int, [c_void_p, P, P, P, P, P]),
    "gm_set_model": (c_int, [c_void_p, c_int, c_int, c_int, c_double, c_int, P, P, P, c_int, P, P,
                             P, P, P, P, P]),
    "gm_model_generation": (c_i64, [c_void_p]),
    "gm_set_dims": (c_int, [c_void_p, c_int, c_int]),
    "gm_set_node_range": (c_int, [c_void_p, c_i64, c_i64]),
    "gm_linearize": (c_int, [c_void_p, c_i64, P, P, P, P, P, P, P, c_void_p]),
    "gm_step": (c_int, [c_void_p, c_i64, P, P, P, c_void_p]),
    "gm_set_linearize_mode": (c_int, [c_void_p, c_int]),
    "gm_trunk_step": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_double, c_double, c_double,
                              c_double, c_double, c_double, P, P, P, c_double, c_int, P, P, P, P,
                              c_void_p]),
    "gm_gamma_ld": (c_int, [c_int, c_int]),
    "gm_condense_gammas": (c_int, [c_void_p, c_int, c_int, P, P, P, P, P, P, c_int, c_void_p]),
    "gm_condense_gammas_stage": (c_int, [c_void_p, c_int, c_int, c_int, P, P, P, P, P, P, c_int,
                                         c_void_p]),
    "gm_condense_cost": (c_int, [c_void_p, c_int, c_int, P, c_int, P, c_i64, P, c_i64, P, c_i64, P,
                                 c_i64, P, P, c_int, c_void_p]),
    "gm_condense_fused": (c_int, [c_void_p, c_int, c_int, P, P, P, P, P, P, c_int, P, c_i64, P,
                                  c_i64, P, c_i64, P, c_i64, P, P, c_void_p]),
    "gm_constraint_rows": (c_int, [c_void_p, c_int, c_int, P, c_int, c_int, P, P, P, c_int, P, P,
                                   P, P, P, P, c_void_p]),
    "gm_node_hessians": (c_int, [c_void_p, c_int, c_int, P, c_int, P, c_i64, P, c_i64, P, P,
                                 c_void_p]),
    "gm_sum_nodes": (c_int, [c_void_p, c_int, c_int, c_int, c_int, P, P, P, c_void_p]),
    "gm_param_count": (c_int, [c_void_p]),
    "gm_loss_gradients": (c_int, [c_void_p, c_int, P, P, P, P, c_double, P, P, c_void_p]),
    "gm_expand_soft": (c_int, [c_void_p, c_int, c_int, c_int, P, P, P, P, c_int, P, P, P, P, P, P,
                               P, c_void_p]),
    "gm_solve_qp": (c_int, [c_void_p, c_int, c_int, c_int, P, P, P, P, P,
                            ctypes.POINTER(QpSettingsC), P, P, P, P, P, c_void_p]),
    "gm_qp_profile": (c_int, [c_int]),
    "gm_qp_phase_cycles": (c_int, [P]),
    "gm_cond_profile": (c_int, [c_int]),
    "gm_cond_phase_cycles": (c_int, [P]),
    "gm_last_condense_kernel": (c_int, [c_void_p]),
    "gm_comm_available": (c_int, []),
    "gm_comm_unique_id": (c_int, [P]),
    "gm_init_comm": (c_int, [c_void_p, P, c_int, c_int]),
    "gm_comm_destroy": (c_int, [c_void_p]),
    "gm_allreduce_sum": (c_int, [c_void_p, P, c_i64, c_void_p]),
    "gm_sendrecv": (c_int, [c_void_p, c_int, P, P, P, c_int, P, P, P, c_void_p]),
    "gm_chol_check": (c_int, [c_void_p, c_int, P, P, P, P, P, c_void_p]),
    "gm_set_condense_mode": (c_int, [c_void_p, c_int]),
    "gm_gram_check": (c_int, [c_void_p, c_int, c_int, P, P, P, c_void_p]),
    "gm_gather_rows": (c_int, [c_void_p, P, P, P, c_int, c_i64, c_i64, c_int, c_i64, c_void_p]),
    "gm_scatter_rows": (c_int, [c_void_p, P, P, P, c_int, c_i64, c_i64, c_int, c_i64, c_void_p]),
    "gm_reconstruct_states": (c_int, [c_void_p, c_int, c_int, P, c_int, P, c_int, P, c_void_p]),
    "gm_mpc_finish": (c_int, [c_void_p, c_int, c_int, P, c_int, P, c_int, P, P, P, P, P, P, c_double,
                              c_int, P, c_int, P, P, P, P, P, P, P, c_void_p]),
    "gm_mpc_finish_rollout": (c_int, [c_void_p, c_int, c_int, P, P, P, P, P, P, c_int, P, P, P, P, P, P,
                                      c_double, c_int, P, c_int, P, P, P, P, P, P, P, c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def lib():
    """Load the library once; raise if it is missing (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"B200 library not built: {LIB_PATH} is missing. Run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (or `make -C "
                    "paper_2602_17601_b200/csrc`). There is no CPU fallback.")
            handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def addr(t) -> int | None:
    """Raw address of a torch tensor / numpy array (None passes NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


class Context:
    """Owns one ``gm_ctx`` (weights, graph tables and scratch on one device)."""

    def __init__(self, device: int):
        self.device = int(device)
        h = c_void_p()
        rc = lib().gm_create(ctypes.byref(h), self.device)
        if rc != GM_OK:
            raise RuntimeError(f"gm_create(device={device}) failed with code {rc} "
                               "(is a CUDA device present?)")
        self.handle = h
        self.graph_key = None
        self.model_key = None
        self.node_range = None

    def close(self):
        if self.handle:
            lib().gm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int, what: str):
        if rc == GM_OK:
            return
        msg = lib().gm_last_error(self.handle)
        msg = msg.decode() if msg else ""
        text = f"{what}: {msg}"
        if rc == GM_ERR_CONFIG:
            raise ConfigurationError(text)
        if rc == GM_ERR_NUMERIC:
            raise FloatingPointError(text)
        raise RuntimeError(text)

    def call(self, name: str, *args):
        self.check(getattr(lib(), name)(self.handle, *args), name)


def require_cuda():
    """The device path needs a CUDA device; fail loudly otherwise."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_17601_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch
