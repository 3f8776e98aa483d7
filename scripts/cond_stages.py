"""Per-stage cycle accounting of the pipelined K-COND (CTA 0) on one cfg4
wave or the cfg5 mesh (diagnostics): python scripts/cond_stages.py [B|mesh].
Needs the library built with the counters compiled in:
    make -C paper_2602_17601_b200/csrc clean && make -C paper_2602_17601_b200/csrc EXTRA=-DGM_COND_PROF"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import _runtime, workloads
from paper_2602_17601_b200.batch import BatchedMpc

N = 20
cfg = pkg.MpcConfig(horizon=N, dt=0.01)
if len(sys.argv) > 1 and sys.argv[1] == "mesh":  # cfg5: 400 x 250 mesh, one instance
    from paper_2602_17601_b200.partition import PartitionedMpc, partition_nodes
    topo, model, states, inputs, spec = workloads.mesh_problem(400, 250, N, 0.01, 0)
    spec.freeze()
    pm = PartitionedMpc(model, topo, spec, cfg, partition_nodes(topo, 1, 0))
    ls = torch.from_numpy(np.ascontiguousarray(np.concatenate([states, states[-1:]], 0))).cuda()
    li = torch.from_numpy(inputs).cuda()
    x0 = torch.from_numpy(np.ascontiguousarray(states[0])).cuda()
    run = lambda: (pm.load(x0, ls, li), pm.enqueue())
else:  # cfg4 wave: B instances of the M=200 chain ("cfg3": one M=1000 chain)
    cfg3 = len(sys.argv) > 1 and sys.argv[1] == "cfg3"
    B = 1 if cfg3 else (int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
    M = 1000 if cfg3 else 200
    topo, model, _, _, spec = workloads.scaling_problem(M, N, 0.01, 0)
    xs, ls, li, xr = [], [], [], []
    for i in range(B):
        st, inp = workloads.batch_instance(i, M, N)
        xs.append(st[0]); ls.append(np.concatenate([st, st[-1:]], 0)); li.append(inp)
        xr.append(np.repeat(st[0][:, None, :], N + 1, axis=1))
    d = [torch.from_numpy(np.stack(v)).cuda() for v in (xs, ls, li, xr)]
    bm = BatchedMpc(model, topo, spec, cfg, B)
    run = lambda: (bm.load(*d), bm.enqueue())
for _ in range(2):
    run()
torch.cuda.synchronize()
L = _runtime.lib()
if L.gm_cond_profile(1) != 0:
    sys.exit("library built without -DGM_COND_PROF (see the docstring)")
run()
torch.cuda.synchronize()
out = np.zeros(768, dtype=np.uint64)
L.gm_cond_phase_cycles(out.ctypes.data)
L.gm_cond_profile(0)
c = out.reshape(32, 24).astype(np.float64)
names = ["R item", "R emptyW", "R flagW", "R tileW", "H fullW", "H busy", "H fold", "items",
         "R in+iss", "R Qs", "R rec", "R w+flag", "H QG+bar", "H rows", "H g", "-", "R cpW", "R barR", "R issue", "R pref", "R fence", "H qg"]
print("per item (cycles), CTA 0; k = stage")
sl = [0, 1, 2, 18, 19, 3, 9, 10, 11, 4, 5, 21, 12, 13, 14, 6, 7]
print("k  " + "".join(f"{names[s]:>9s}" for s in sl))
for k in range(32):
    if c[k, 7] == 0:
        continue
    it = c[k, 7]
    print(f"{k:<3d}" + "".join(f"{c[k, s] / (it if s != 7 else 1):9.0f}" for s in sl))
