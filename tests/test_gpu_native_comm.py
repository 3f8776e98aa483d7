"""Native data plane (gm_init_comm / gm_sendrecv / gm_allreduce_sum; SURVEY
8b, 8e) on the one GPU of the test box: a world-1 NCCL communicator, byte
transfers to self, the fp64 all-reduce, all stream-ordered and inside a
captured CUDA graph; and the partitioned step driven through it, eager and
captured, against the oracle.  World > 1 needs one GPU per rank (NCCL
rejects two ranks on one device); the exchange logic itself is covered by
the LocalTransport GPU tests and the gloo CPU tests."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def transport():
    import torch

    from paper_2602_17601_b200.partition import NcclTransport

    tr = NcclTransport(0, 1, torch.device("cuda", 0), unique_id=NcclTransport.unique_id())
    yield tr
    tr.close()


def test_comm_available_and_errors():
    import ctypes

    from paper_2602_17601_b200._runtime import Context, lib

    assert lib().gm_comm_available() == 1
    ctx = Context(0)
    try:
        with pytest.raises(Exception):  # no communicator yet
            ctx.call("gm_allreduce_sum", None, 0, None)
        buf = (ctypes.c_uint8 * 128)()
        with pytest.raises(Exception):  # rank outside the world
            ctx.call("gm_init_comm", ctypes.addressof(buf), 1, 1)
    finally:
        ctx.close()


def test_sendrecv_self_and_allreduce(transport):
    import torch

    dev = torch.device("cuda", 0)
    a = torch.arange(1000, dtype=torch.float32, device=dev)
    b = torch.zeros(1000, dtype=torch.float32, device=dev)
    transport.sendrecv({0: a}, {0: b})
    x = torch.linspace(-1, 1, 777, dtype=torch.float64, device=dev)
    y = x.clone()
    transport.allreduce_sum(y)  # world 1: the identity
    outs = [torch.empty_like(x)]
    transport.all_gather(outs, x)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(x, y) and torch.equal(outs[0], x)
    with pytest.raises(ValueError):
        transport.allreduce_sum(a)  # fp64 only


def test_exchange_inside_cuda_graph(transport):
    """gather kernel -> NCCL send/recv -> scatter kernel -> all-reduce, captured
    once and replayed with new data."""
    import torch

    from paper_2602_17601_b200.device import engine
    from paper_2602_17601_b200.graph import chain_topology

    dev = torch.device("cuda", 0)
    eng = engine(chain_topology(16))
    ld = 32
    W = torch.randn(16, 6, ld, device=dev)
    idx = torch.tensor([3, 7, 11], dtype=torch.int32, device=dev)
    dst_idx = torch.tensor([0, 1, 2], dtype=torch.int32, device=dev)
    sbuf = torch.empty(3, 6, ld, device=dev)
    rbuf = torch.empty(3, 6, ld, device=dev)
    out = torch.zeros(16, 6, ld, device=dev)
    red = torch.zeros(64, dtype=torch.float64, device=dev)

    def step():
        sp = eng.stream_ptr()
        rb = 6 * ld * 4  # one node's 6 rows of fp32
        eng.ctx.call("gm_gather_rows", W.data_ptr(), sbuf.data_ptr(), idx.data_ptr(), 3, rb, rb, 1, 0, sp)
        transport.sendrecv({0: sbuf}, {0: rbuf})
        eng.ctx.call("gm_scatter_rows", rbuf.data_ptr(), out.data_ptr(), dst_idx.data_ptr(), 3, rb, rb, 1, 0,
                     sp)
        red.copy_(W[:, 0, :4].reshape(-1).double())
        transport.allreduce_sum(red)

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(2):
        W.copy_(torch.randn_like(W))
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out[:3], W[idx.long()])
        assert torch.equal(red, W[:, 0, :4].reshape(-1).double())


def test_partitioned_step_native_transport_graph(transport):
    """PartitionedMpc with the native transport: eager step, captured step
    (one CUDA graph per RTI step) and the oracle agree."""
    from oracle import ref_port as O
    from paper_2602_17601_b200 import MpcConfig, workloads
    from paper_2602_17601_b200.partition import PartitionedMpc, partition_nodes

    N = 6
    topo, model, states, inputs, spec = workloads.mesh_problem(12, 10, N, 0.01, 2)
    cfg = MpcConfig(horizon=N, dt=0.01)
    part = partition_nodes(topo, 1, 0)
    pm = PartitionedMpc(model, topo, spec, cfg, part, transport=transport)
    ls = np.concatenate([states, states[-1:]], 0)
    u_e, st_e, it_e = pm.step(states[0], ls, inputs)
    nxt_e = pm.next_states.cpu().numpy().copy()
    u_g, st_g, it_g = pm.step_graph(states[0], ls, inputs)
    nxt_g = pm.next_states.cpu().numpy().copy()
    u_g2, _, _ = pm.step_graph(states[0], ls, inputs)  # replay of the cached graph
    assert np.array_equal(u_e, u_g) and np.array_equal(u_g, u_g2)
    assert (st_e, it_e) == (st_g, it_g)
    assert np.array_equal(nxt_e, nxt_g)
    ref = O.mpc_step(model, topo, spec, states[0], ls, inputs, N)
    from paper_2602_17601_b200.qpsolver import STATUS_BY_CODE

    assert STATUS_BY_CODE[st_e].value == ref["status"]
    assert np.max(np.abs(u_e - ref["u_applied"])) / max(1.0, np.max(np.abs(ref["u_applied"]))) <= 1e-4


def test_capture_requires_stream_ordered_transport():
    """A world > 1 step can only be captured with the native transport: the
    in-process / torch.distributed transports wait on the host."""
    from paper_2602_17601_b200 import MpcConfig, workloads
    from paper_2602_17601_b200.errors import ConfigurationError
    from paper_2602_17601_b200.partition import LocalHub, LocalTransport, PartitionedMpc, partition_nodes

    N = 4
    topo, model, states, inputs, spec = workloads.mesh_problem(6, 5, N, 0.01, 2)
    part = partition_nodes(topo, 2, 0)
    pm = PartitionedMpc(model, topo, spec, MpcConfig(horizon=N, dt=0.01), part,
                        transport=LocalTransport(LocalHub(2), 0))
    with pytest.raises(ConfigurationError):
        pm.capture()
