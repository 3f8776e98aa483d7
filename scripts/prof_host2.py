"""Host-side cost of the pieces of mpc_step at cfg3 (graph replay, copies)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads, mpc as mpcmod
topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
x = pkg.SystemState(states[0])
st = pkg.mpc_init(x, cfg, 6)
for _ in range(5):
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
torch.cuda.synchronize()
eng = pkg.device.engine(topo, model)
plan = [v for k, v in eng.cache.items() if isinstance(k, tuple) and k[0] == "plan"][0]
print("graph nodes:", plan.graph is not None)
g = plan.graph
t0 = time.perf_counter(); 
for _ in range(20): g.replay()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"replay call {1e3*(t1-t0)/20:.3f} ms, +drain {1e3*(t2-t1):.2f} ms for 20")
a = torch.empty((21, 1000, 6), dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(100): a.copy_(b)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"D2D copy_ call {1e3*(t1-t0)/100:.4f} ms")
o = plan.outbuf
t0 = time.perf_counter()
for _ in range(100): c = o.clone()
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"clone call {1e3*(t1-t0)/100:.4f} ms, outbuf {o.numel()*8/1e6:.2f} MB")
for _ in range(3):
    t0 = time.perf_counter(); u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg); t1 = time.perf_counter()
    print(f"mpc_step wall {1e3*(t1-t0):.3f} ms, device stages {st1.last_timing.linearize_ms + st1.last_timing.condense_ms + st1.last_timing.solve_ms:.3f}")
