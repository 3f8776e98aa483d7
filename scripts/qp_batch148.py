"""148 copies of the cfg3 QP in one K-QP launch (one per SM): enough
samples for a source-level ncu view of the solver (diagnostics)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads
from paper_2602_17601_b200.qpsolver import solve_qp_batched
from oracle import ref_port as O

topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
lin = O.linearize_trajectory(model, topo, states, inputs)
q = O.condense_ocp(spec, lin, states[0])
H, g, C, d, _ = O.expand_soft_constraints(q)
B = 148
sols = solve_qp_batched(np.stack([H] * B), np.stack([g] * B), np.stack([C] * B), np.stack([d] * B))
sols = solve_qp_batched(np.stack([H] * B), np.stack([g] * B), np.stack([C] * B), np.stack([d] * B))
print(sols[0].status, sols[0].iterations)
