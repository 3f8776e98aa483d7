"""Solve one QP (a golden fixture's expanded QP) -- for profiling K-QP alone."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_17601_b200 as pkg
from tests.golden_io import load
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1_chain10"
d = load(name)
p = pkg.QpProblem(d["x_H"], d["x_g"], d["x_C"], d["x_d"])
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    s = pkg.solve_qp(p)
print(s.status, s.iterations, float(np.max(np.abs(s.u - d["sol_u"]))))
