"""Per-phase cycle breakdown of K-QP on a fixture QP (diagnostics).  Needs the
library built with the counters: `make -C paper_2602_17601_b200/csrc
EXTRA=-DGM_QP_PROF` (touch k_qp.cu first); gm_qp_profile fails otherwise."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import _runtime
from tests.golden_io import load
names = ["setup", "residuals", "tests+best", "w+build_k", "cholesky", "inv_diag", "rp/mu+aff_rhs",
         "kkt(excl solve)", "steps/sigma", "update", "pre-solve", "chol_solve",
         "[res] h_apply", "[res] ct+c_apply+loops / [bk] w,kee,wg", "[bk] tiles", "[bk] diag"]
if "--chol" in sys.argv:  # slots 13-15: the Cholesky pivot chain (warp 0)
    names[13:16] = ["[chol] look-ahead wait", "[chol] panel + E", "[chol] factor8 + publish"]
for case in [a for a in sys.argv[1:] if not a.startswith("--")] or ["cfg1_chain10"]:
    if case == "cfg3":
        from paper_2602_17601_b200 import workloads
        from oracle import ref_port as O
        topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
        lin = O.linearize_trajectory(model, topo, states, inputs)
        q = O.condense_ocp(spec, lin, states[0])
        H, g, C, d, _ = O.expand_soft_constraints(q)
    else:
        dd = load(case); H, g, C, d = dd["x_H"], dd["x_g"], dd["x_C"], dd["x_d"]
    p = pkg.QpProblem(H, g, C, d)
    s = pkg.solve_qp(p)
    L = _runtime.lib()
    if L.gm_qp_profile(2 if "--chol" in sys.argv else 1) != 0:
        sys.exit("qp_phases: library built without -DGM_QP_PROF")
    s = pkg.solve_qp(p)
    out = np.zeros(16, dtype=np.uint64)
    L.gm_qp_phase_cycles(out.ctypes.data)
    L.gm_qp_profile(0)
    tot = out[:12].sum()
    print(f"{case}: n={p.n} m={p.m} iters={s.iterations} total={tot} cycles ({tot/1.96e3:.0f} us @1.96GHz), per-iter {tot/max(1,s.iterations):.0f}")
    for i, nm in enumerate(names):
        if out[i]:
            print(f"   {nm:18s} {int(out[i]):10d}  {100*out[i]/tot:5.1f}%  per-iter {out[i]/max(1,s.iterations):9.0f}  per-step {out[i]/max(1,s.iterations)/(p.n/2):7.0f}")
