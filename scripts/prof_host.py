"""Host-side profile of the public mpc_step at cfg3 (where the e2e - device gap goes)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads
topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
x = pkg.SystemState(states[0])
st = pkg.mpc_init(x, cfg, 6)
for _ in range(5):
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
t1 = time.perf_counter()
print(f"wall per step {1e3*(t1-t0)/50:.3f} ms; device stages {st1.last_timing}")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
