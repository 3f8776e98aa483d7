"""Diagnostic: where the u error at the 100x100 mesh comes from (condensing
fp32 vs QP), printed as relative errors."""
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import ref_port as O
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads
from paper_2602_17601_b200.condensing import OcpSpec
R, C = (int(v) for v in sys.argv[1:3])
topo, model, states, inputs, spec = workloads.mesh_problem(R, C, 20, 0.01, 0)
lin = O.linearize_trajectory(model, topo, states, inputs)
gu, gx = O.condense_gammas(lin, states[0], threads=8)
linb = pkg.linearize_trajectory(model, topo, states, inputs)
gub, gxb = pkg.condense_gammas(linb, states[0])
rel = lambda a, b: float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))
print("a_self", rel(linb.a_self, lin.a_self), "a_nbr", rel(linb.a_nbr, lin.a_nbr), "b", rel(linb.b, lin.b))
print("gu", rel(gub, gu), "gx", rel(gxb, gx))
for rs in (0.01, 1.0):
    sp = OcpSpec(topo, 20, spec.q, spec.x_ref, np.tile(np.eye(6) * rs, (20, 1, 1)), spec.u_ref,
                 spec.input_constraints, spec.state_constraints)
    q = O.condense_ocp(sp, lin, states[0], gammas=(gu, gx), threads=8)
    qb = pkg.condense_ocp(sp, linb, states[0], gammas=(gub, gxb))
    H, g, Cc, d, n0 = O.expand_soft_constraints(q)
    Hb, gb, Cb, db, _ = O.expand_soft_constraints(qb)
    warm = np.zeros(H.shape[0]); warm[:n0] = inputs.reshape(-1)
    s = O.solve_qp(H, g, Cc, d, warm_start=warm)
    sb = O.solve_qp(Hb, gb, Cb, db, warm_start=warm)   # oracle QP on GPU-condensed data
    sg = pkg.solve_qp(pkg.QpProblem(Hb, gb, Cb, db), pkg.SolverSettings(warm_start=warm))
    sc = max(1.0, np.max(np.abs(s.u[:n0])))
    print(f"R={rs}: H {rel(qb.h, q.h):.2e} g {rel(qb.g, q.g):.2e} C {rel(qb.c, q.c):.2e} cond {np.linalg.cond(q.h):.3g} "
          f"| u_all(oracleQP on gpu H) {np.max(np.abs(sb.u[:n0]-s.u[:n0]))/sc:.2e} u0 {np.max(np.abs(sb.u[:6]-s.u[:6]))/sc:.2e} "
          f"| gpuQP vs oracleQP same data {np.max(np.abs(sg.u[:n0]-sb.u[:n0]))/sc:.2e} it {s.iterations} {sb.iterations} {sg.iterations}")
