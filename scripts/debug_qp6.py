import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2602_17601_b200 as pkg
from tests.golden_io import random_qps
from oracle import ref_port as O
q = random_qps()[6]
print("H eig", np.linalg.eigvalsh(q.H)[:3], "C", q.C, "d", q.d)
for k in range(0, 7):
    s = pkg.solve_qp(pkg.QpProblem(q.H, q.g, q.C, q.d), pkg.SolverSettings(max_iterations=k))
    r = O.solve_qp(q.H, q.g, q.C, q.d, max_iterations=k)
    print(k, s.status.value, s.iterations, np.round(s.u, 6), "| ref", r.status, r.iterations, np.round(r.u, 6), s.stationarity, r.stationarity)
