"""Where the cfg3 end-to-end time beyond the device step goes: host time
before the step graph's launch, launch -> synchronize return, after it."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads

topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze(); model.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
dev = torch.device("cuda", 0)
state = pkg.MpcState(lin_states=torch.from_numpy(np.tile(states[0], (21, 1, 1))).to(dev),
                     lin_inputs=torch.zeros((20, 6), dtype=torch.float64, device=dev))
xs = pkg.SystemState(states[0])
marks = {}
orig_replay = torch.cuda.CUDAGraph.replay
orig_sync = torch.cuda.Stream.synchronize
def replay(self):
    marks["pre"] = time.perf_counter()
    orig_replay(self)
    marks["launched"] = time.perf_counter()
def sync(self):
    orig_sync(self)
    marks["synced"] = time.perf_counter()
torch.cuda.CUDAGraph.replay = replay
torch.cuda.Stream.synchronize = sync
for _ in range(20):
    u, state = pkg.mpc_step(model, topo, spec, xs, state, cfg)
torch.cuda.synchronize()
acc = np.zeros(4); n = 300
for _ in range(n):
    t0 = time.perf_counter()
    u, state = pkg.mpc_step(model, topo, spec, xs, state, cfg)
    t1 = time.perf_counter()
    acc += [marks["pre"] - t0, marks["launched"] - marks["pre"], marks["synced"] - marks["launched"], t1 - marks["synced"]]
acc = acc / n * 1e3
print("ms per step: prologue %.3f | launch %.3f | launch->synced %.3f | epilogue %.3f | total %.3f" % (*acc, acc.sum()))
