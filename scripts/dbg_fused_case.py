import sys
sys.path.insert(0, ".")
from tests.test_gpu_fused import _run, _check
from paper_2602_17601_b200.graph import chain_topology, mesh_topology
M, N, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
topo = chain_topology(M) if sys.argv[4] == "chain" else mesh_topology(23, 17)
ref, outs = _run(topo, N, 6, 6, B, seed=11, reps=1, mode=0)
_check(ref, outs, N * 6, 6, N, tol=1e-5)
print("ok")
