"""Solve the cfg3 expanded QP once (profiling K-QP at n=140, m=280)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads
from oracle import ref_port as O
topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
lin = O.linearize_trajectory(model, topo, states, inputs)
q = O.condense_ocp(spec, lin, states[0])
H, g, C, d, _ = O.expand_soft_constraints(q)
p = pkg.QpProblem(H, g, C, d)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    s = pkg.solve_qp(p)
print(s.status, s.iterations)
