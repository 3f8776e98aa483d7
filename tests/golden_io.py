"""Load the golden fixtures (made by oracle/make_golden.py from the reference)
back into model / topology / spec objects of the product package (pure data
types), so the same fixture drives both the oracle and the GPU path."""

from __future__ import annotations

from pathlib import Path
from types import SimpleNamespace

import numpy as np

from paper_2602_17601_b200.condensing import OcpSpec, StateConstraint
from paper_2602_17601_b200.gnn import GnnModel, LinearizedDynamics, Normalization
from paper_2602_17601_b200.graph import GraphTopology, chain_topology, mesh_topology
from paper_2602_17601_b200.mlp import MlpParams

DIR = Path(__file__).resolve().parent / "golden"
STATUS = ("optimal", "max_iterations", "primal_infeasible", "numerical_failure")


def load(name: str):
    with np.load(DIR / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def model_from(d, prefix=""):
    def mlp(name):
        dims = [int(v) for v in d[f"{prefix}{name}_dims"]]
        L = len(dims) - 1
        return MlpParams(dims, [d[f"{prefix}{name}_W{l}"] for l in range(L)],
                         [d[f"{prefix}{name}_b{l}"] for l in range(L)])

    dt, n_p, n_u, n_m = d[f"{prefix}meta"]
    n_p, n_u, n_m = int(n_p), int(n_u), int(n_m)
    nx = 2 * n_p
    nrm = d[f"{prefix}norm"]
    norm = Normalization(nrm[:nx], nrm[nx:2 * nx], nrm[2 * nx:2 * nx + n_u], nrm[2 * nx + n_u:])
    return GnnModel(mlp("psi"), mlp("phi"), float(dt), n_p, n_u, n_m, norm)


def topo_from_ptr(ptr, lst, bound=None):
    M = len(ptr) - 1
    nbrs = tuple(tuple(int(v) for v in lst[ptr[i]:ptr[i + 1]]) for i in range(M))
    if bound is None:
        bound = max(1, max((len(n) for n in nbrs), default=1))
    return GraphTopology(M, nbrs, int(bound))


def spec_from(d, topo, prefix=""):
    q, x_ref, r, u_ref = (d[prefix + k] for k in ("q", "x_ref", "r", "u_ref"))
    icons = None
    if prefix + "icons_C" in d:
        icons = [(C, dd) for C, dd in zip(d[prefix + "icons_C"], d[prefix + "icons_d"])]
    scons = []
    meta = d[prefix + "scons_meta"]
    cc, dd = d[prefix + "scons_c"], d[prefix + "scons_d"]
    row = 0
    for node, stage, soft, rho1, rho2, rows in meta:
        rows = int(rows)
        scons.append(StateConstraint(int(node), int(stage), cc[row:row + rows], dd[row:row + rows],
                                     soft=bool(soft), rho1=float(rho1), rho2=float(rho2)))
        row += rows
    return OcpSpec(topo, q.shape[1] - 1, q, x_ref, r, u_ref, icons, scons)


def pipeline_case(name):
    """A full-pipeline fixture (cfg1 / P3 / P4 chains, mesh6x5 / mesh_p3
    4-neighbour grids) as objects + expected arrays."""
    d = load(name)
    model = model_from(d)
    M = d["states"].shape[1]
    topo = mesh_topology(*(int(v) for v in d["mesh"])) if "mesh" in d else chain_topology(M)
    spec = spec_from(d, topo)
    return SimpleNamespace(d=d, model=model, topo=topo, spec=spec, states=d["states"],
                           inputs=d["inputs"], x0=d["states"][0])


def random_condense_cases():
    d = load("p2_random_condense")
    out = []
    t = 0
    while f"c{t}_a_self" in d:
        p = f"c{t}_"
        topo = topo_from_ptr(d[p + "nbr_ptr"], d[p + "nbr_list"], 2)
        N = d[p + "a_self"].shape[0]
        lin = LinearizedDynamics(topo, N, d[p + "a_self"], d[p + "a_nbr"], d[p + "b"], d[p + "c"])
        spec = spec_from(d, topo, p)
        out.append(SimpleNamespace(topo=topo, lin=lin, spec=spec, x0=d[p + "x0"],
                                   gamma_u=d[p + "gamma_u"], gamma_x=d[p + "gamma_x"],
                                   qp={k: d[p + "qp_" + k] for k in ("h", "g", "c", "d", "soft")}))
        t += 1
    return out


def random_qps():
    d = load("qp_random")
    out = []
    t = 0
    while f"q{t}_H" in d:
        p = f"q{t}_"
        out.append(SimpleNamespace(H=d[p + "H"], g=d[p + "g"], C=d[p + "C"], d=d[p + "d"],
                                   u=d[p + "u"], duals=d[p + "duals"],
                                   status=STATUS[int(d[p + "meta"][0])],
                                   iterations=int(d[p + "meta"][1])))
        t += 1
    return out


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def mpc_branch_cases():
    """mpc_step sequences of the reference under non-default MpcConfig
    branches (oracle/make_golden.py round2): returns (model, topo, spec,
    bad_spec, x_seq, {case: [step dicts]})."""
    d = load("mpc_branches")
    model = model_from(d)
    M = d["states"].shape[1]
    topo = chain_topology(M)
    spec = spec_from(d, topo)
    bad = OcpSpec(topo, spec.horizon, spec.q, spec.x_ref, spec.r, spec.u_ref,
                  spec.input_constraints,
                  list(spec.state_constraints) + [StateConstraint(0, 1, d["bad_row_c"], d["bad_row_d"])])
    cases = {}
    for c in d["cases"]:
        c = str(c)
        steps = []
        for t in range(int(d[c + "_steps"])):
            p = f"{c}_{t}_"
            steps.append({k: d[p + k] for k in ("u", "lin_states", "lin_inputs", "planned_states",
                                                "planned_inputs", "last_applied", "filtered", "meta")})
        cases[c] = steps
    return SimpleNamespace(model=model, topo=topo, spec=spec, bad=bad, x_seq=d["x_seq"], cases=cases)


def qp_round2():
    d = load("qp_round2")

    def get(prefix):
        out, t = [], 0
        while f"{prefix}{t}_H" in d:
            p = f"{prefix}{t}_"
            out.append(SimpleNamespace(H=d[p + "H"], g=d[p + "g"], C=d[p + "C"], d=d[p + "d"],
                                       u=d[p + "u"], duals=d[p + "duals"],
                                       status=STATUS[int(d[p + "meta"][0])],
                                       iterations=int(d[p + "meta"][1]),
                                       cap=int(d[p + "meta"][2]) if d[p + "meta"].size > 2 else 50))
            t += 1
        return out

    return SimpleNamespace(cap=get("cap"), batch=get("b"), infeas_u=d["infeas_u"],
                           infeas_status=STATUS[int(d["infeas_meta"][0])],
                           infeas_iterations=int(d["infeas_meta"][1]),
                           infeas_primal=float(d["infeas_meta"][2]))


def local_condense_cases():
    """Reference condense_local / assemble_qp outputs (oracle/make_golden.py
    local_condense)."""
    d = load("local_condense")
    out, t = [], 0
    while f"c{t}_a_self" in d:
        p = f"c{t}_"
        topo = topo_from_ptr(d[p + "nbr_ptr"], d[p + "nbr_list"], 2)
        N = d[p + "a_self"].shape[0]
        lin = LinearizedDynamics(topo, N, d[p + "a_self"], d[p + "a_nbr"], d[p + "b"], d[p + "c"])
        out.append(SimpleNamespace(
            topo=topo, lin=lin, spec=spec_from(d, topo, p), x0=d[p + "x0"], h=d[p + "h"],
            g=d[p + "g"], rows=d[p + "rows"], c_rows=d[p + "c_rows"], d_rows=d[p + "d_rows"],
            qa={k: d[p + "qa_" + k] for k in ("h", "g", "c", "d", "soft", "rho1", "rho2")},
            lhg_h=d[p + "lhg_h"], lhg_g=d[p + "lhg_g"]))
        t += 1
    return out


def training_cases():
    """Reference loss_gradients outputs (oracle/make_golden.py training_grads)."""
    d = load("training_grads")
    out = []
    for name in d["cases"]:
        p = str(name) + "_"
        topo = topo_from_ptr(d[p + "nbr_ptr"], d[p + "nbr_list"])
        out.append(SimpleNamespace(name=str(name), topo=topo, model=model_from(d, p + "m_"),
                                   X=d[p + "X"], U=d[p + "U"], Xn=d[p + "Xn"], W=d[p + "W"],
                                   lam=float(d[p + "lam"]), loss=float(d[p + "loss"]),
                                   grads=d[p + "grads"]))
    return out
