"""cProfile of the public mpc_step at cfg3 (host-side overhead around the step
graph; diagnostics)."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads

topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze()
model.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
dev = torch.device("cuda", 0)
state = pkg.MpcState(lin_states=torch.from_numpy(np.tile(states[0], (21, 1, 1))).to(dev),
                     lin_inputs=torch.zeros((20, 6), dtype=torch.float64, device=dev))
xs = pkg.SystemState(states[0])
for _ in range(10):
    u, state = pkg.mpc_step(model, topo, spec, xs, state, cfg)
torch.cuda.synchronize()


def run(n=300):
    global state
    for _ in range(n):
        _, state = pkg.mpc_step(model, topo, spec, xs, state, cfg)


pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
