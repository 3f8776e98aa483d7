"""Host-side profile of the public mpc_step at cfg3 (where the e2e time
beyond the device step goes)."""
import cProfile, pstats, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads
topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
xs = pkg.SystemState(states[0])
dev = torch.device("cuda", 0)
st0 = pkg.MpcState(lin_states=torch.from_numpy(np.tile(states[0], (21, 1, 1))).to(dev),
                   lin_inputs=torch.zeros((20, 6), dtype=torch.float64, device=dev))
for _ in range(10):
    pkg.mpc_step(model, topo, spec, xs, st0, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    pkg.mpc_step(model, topo, spec, xs, st0, cfg)
print("e2e ms", (time.perf_counter() - t0) * 10)
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    pkg.mpc_step(model, topo, spec, xs, st0, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
