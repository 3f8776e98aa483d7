"""The C ABI library: loads without a GPU, exports every symbol the header
declares, and its host-side graph index construction is bit-exact with the
reference tables (gnn.py:107-126, condensing.py:158-172).  CPU only: no
device compute is called here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2602_17601_b200 import _runtime
from paper_2602_17601_b200.errors import ConfigurationError
from tests.golden_io import load

HEADER = Path(__file__).resolve().parents[1] / "include" / "gnnmpc_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gm_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _runtime.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes binding covers exactly the declared entry points
    assert sorted(_runtime.EXPORTED_SYMBOLS) == syms
    assert lib.gm_abi_version() == 1


class HostCtx:
    def __init__(self):
        h = ctypes.c_void_p()
        assert _runtime.lib().gm_create(ctypes.byref(h), -1) == 0
        self.h = h

    def __del__(self):
        _runtime.lib().gm_destroy(self.h)

    def set_graph(self, ptr, lst, bound):
        ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        lst = np.ascontiguousarray(lst, dtype=np.int64)
        rc = _runtime.lib().gm_set_graph(self.h, len(ptr) - 1, int(bound), ptr.ctypes.data,
                                         lst.ctypes.data if lst.size else None)
        return rc, _runtime.lib().gm_last_error(self.h).decode()


def test_graph_tables_bit_exact():
    d = load("graph_tables")
    names = sorted({k[: -len("_nbr_ptr")] for k in d if k.endswith("_nbr_ptr")})
    for name in names:
        ctx = HostCtx()
        rc, msg = ctx.set_graph(d[name + "_nbr_ptr"], d[name + "_nbr_list"], d[name + "_bound"])
        assert rc == 0, msg
        L = _runtime.lib()
        E = int(L.gm_edge_count(ctx.h))
        dm = int(L.gm_max_degree(ctx.h))
        M = len(d[name + "_nbr_ptr"]) - 1
        dst, src = np.empty(E, np.int64), np.empty(E, np.int64)
        gather = np.empty((M, max(dm, 1)), np.int64)
        slots = np.empty((M, 1 + dm), np.int64)
        es = np.empty(E, np.int64)
        rc = L.gm_graph_tables(ctx.h, dst.ctypes.data, src.ctypes.data, gather.ctypes.data,
                               slots.ctypes.data, es.ctypes.data)
        assert rc == 0
        assert np.array_equal(dst, d[name + "_dst"]), name
        assert np.array_equal(src, d[name + "_src"]), name
        assert np.array_equal(gather, d[name + "_gather"]), name
        assert np.array_equal(slots, d[name + "_nbr_idx"]), name
        assert np.array_equal(es, d[name + "_edge_slot"]), name
        assert np.array_equal(np.stack([dst, src], 1).reshape(-1, 2), d[name + "_edges"]), name


@pytest.mark.parametrize("nbrs,bound,needle", [
    (((1, 1), ()), 2, "duplicate"),
    (((0,), ()), 2, "itself"),
    (((5,), ()), 2, "out-of-range"),
    (((1,), (0,)), 0, "neighbor_bound"),
    (((1,), (0,)), 1, None),
    (((1, 0),), 1, "neighbors > bound"),
])
def test_graph_validation_mirrors_reference(nbrs, bound, needle):
    """GraphTopology.__post_init__ rules (graph.py:35-54) enforced natively."""
    ptr = np.concatenate([[0], np.cumsum([len(n) for n in nbrs])])
    lst = np.array([j for n in nbrs for j in n], dtype=np.int64)
    rc, msg = HostCtx().set_graph(ptr, lst, bound)
    if needle is None:
        assert rc == 0
    else:
        assert rc == _runtime.GM_ERR_CONFIG and needle in msg, msg


def test_device_entry_points_refuse_host_context():
    ctx = HostCtx()
    rc, _ = ctx.set_graph([0, 1, 2], [1, 0], 1)
    assert rc == 0
    L = _runtime.lib()
    rc = L.gm_linearize(ctx.h, 1, None, None, None, None, None, None, None, None)
    assert rc != 0
    assert L.gm_gamma_ld(20, 6) == 128 and L.gm_gamma_ld(10, 6) == 64


def test_error_mapping():
    class Fake:
        handle = None

    c = _runtime.Context.__new__(_runtime.Context)
    c.handle = ctypes.c_void_p()
    with pytest.raises(ConfigurationError):
        c.check(_runtime.GM_ERR_CONFIG, "x")
    with pytest.raises(FloatingPointError):
        c.check(_runtime.GM_ERR_NUMERIC, "x")
    with pytest.raises(RuntimeError):
        c.check(_runtime.GM_ERR_CUDA, "x")


def test_frozen_model_is_immutable():
    """GnnModel.freeze (the engine then checks the model by identity instead
    of re-hashing its parameters per step): arrays read-only, layer lists
    tuples, copies unfrozen."""
    import numpy as np
    import pytest

    import paper_2602_17601_b200 as pkg

    m = pkg.init_model(3, 6, 0.01, np.random.default_rng(0)).freeze()
    with pytest.raises(ValueError):
        m.psi.weights[0][0, 0] = 1.0
    with pytest.raises(TypeError):
        m.phi.weights[0] = np.zeros_like(m.phi.weights[0])
    c = m.copy()
    c.psi.weights[0][0, 0] = 1.0
    assert not hasattr(c, "_frozen")


def test_native_comm_entry_points_on_cpu():
    """The native data plane resolves NCCL at run time (no link-time
    dependency): availability, a unique id, and loud errors on a context
    without a communicator or with bad arguments -- none needs a GPU."""
    import ctypes

    from paper_2602_17601_b200._runtime import lib

    L = lib()
    if not L.gm_comm_available():
        pytest.skip("libnccl.so.2 not present in this image")
    a, b = (ctypes.c_uint8 * 128)(), (ctypes.c_uint8 * 128)()
    assert L.gm_comm_unique_id(ctypes.addressof(a)) == 0
    assert L.gm_comm_unique_id(ctypes.addressof(b)) == 0
    assert bytes(a) != bytes(b)  # fresh ids
    assert L.gm_comm_unique_id(None) != 0
    assert L.gm_comm_destroy(None) != 0


def test_qp_phase_counters_are_opt_in():
    """The K-QP per-phase counters cost instruction-cache footprint in the IPM
    loop, so the product build leaves them out: enabling them fails loudly
    (GM_ERR_CONFIG) unless the library was built with -DGM_QP_PROF."""
    from paper_2602_17601_b200._runtime import GM_ERR_CONFIG, lib

    assert lib().gm_qp_profile(1) == GM_ERR_CONFIG
    assert lib().gm_qp_profile(2) == GM_ERR_CONFIG
