"""Per-stage device timings of the public mpc_step at a given workload."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2602_17601_b200 as pkg  # noqa: E402
from paper_2602_17601_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=1000)
ap.add_argument("--N", type=int, default=20)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

topo, model, states, inputs, spec = workloads.scaling_problem(a.M, a.N, 0.01, 0)
spec.freeze()
cfg = pkg.MpcConfig(horizon=a.N, dt=0.01)
x = pkg.SystemState(states[0])
st = pkg.mpc_init(x, cfg, 6)
for r in range(a.reps):
    t0 = time.perf_counter()
    u, st1 = pkg.mpc_step(model, topo, spec, x, st, cfg)
    t1 = time.perf_counter()
    tm = st1.last_timing
    print(f"rep {r}: wall {1e3*(t1-t0):8.3f} ms | lin {tm.linearize_ms:7.3f} cond {tm.condense_ms:7.3f} "
          f"qp {tm.solve_ms:8.3f} ms | status {st1.last_status.value} iters {st1.last_iterations}")
