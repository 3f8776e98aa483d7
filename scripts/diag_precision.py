"""Diagnostic: error budget of the fp32 stages at a large mesh for each
kernel variant (linearize mode 2 = tcgen05 3xTF32 Jacobians, 4 = SIMT fp32;
condense mode 1 = SIMT H, 3 = tcgen05 3xTF32 H), relative to the oracle."""
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import ref_port as O
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads, device
R, C = (int(v) for v in sys.argv[1:3])
topo, model, states, inputs, spec = workloads.mesh_problem(R, C, 20, 0.01, 0)
lin = O.linearize_trajectory(model, topo, states, inputs)
gu, gx = O.condense_gammas(lin, states[0], threads=8)
q = O.condense_ocp(spec, lin, states[0], gammas=(gu, gx), threads=8)
H, g, Cc, d, n0 = O.expand_soft_constraints(q)
warm = np.zeros(H.shape[0]); warm[:n0] = inputs.reshape(-1)
s = O.solve_qp(H, g, Cc, d, warm_start=warm)
rel = lambda a, b: float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))
ctx = device.engine(topo, model).ctx
for lm in (2, 4):
    ctx.call("gm_set_linearize_mode", lm)
    linb = pkg.linearize_trajectory(model, topo, states, inputs)
    ctx.call("gm_set_linearize_mode", 0)
    blk = max(rel(linb.a_self, lin.a_self), rel(linb.a_nbr, lin.a_nbr), rel(linb.b, lin.b))
    for cm in (1, 3):
        ctx.call("gm_set_condense_mode", cm)
        gub, gxb = pkg.condense_gammas(linb, states[0])
        qb = pkg.condense_ocp(spec, linb, states[0])
        ctx.call("gm_set_condense_mode", 0)
        Hb, gb, Cb, db, _ = O.expand_soft_constraints(qb)
        sb = O.solve_qp(Hb, gb, Cb, db, warm_start=warm)
        sc = max(1.0, np.max(np.abs(s.u[:n0])))
        print(f"lin{lm} cond{cm}: blocks {blk:.2e} gu {rel(gub, gu):.2e} H {rel(qb.h, q.h):.2e} g {rel(qb.g, q.g):.2e} "
              f"u_all {np.max(np.abs(sb.u[:n0]-s.u[:n0]))/sc:.2e} u0 {np.max(np.abs(sb.u[:6]-s.u[:6]))/sc:.2e}", flush=True)
