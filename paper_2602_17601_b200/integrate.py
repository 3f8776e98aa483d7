"""Route the UNMODIFIED reference ``gnnmpc.mpc.mpc_step`` through the B200 path.

The reference's ``mpc_step`` (``mpc.py:102-200``) calls its stages through
module globals of ``gnnmpc.mpc`` (hard imports, ``mpc.py:18-21``): stage 1 via
``linearize_trajectory`` inside ``_as_linearizer`` (``:82-87``) -- or any
``Linearizer`` callable passed as ``model`` (``:23``) -- and stages 2-4 via
``condense_gammas``, ``condense_ocp``, ``expand_soft_constraints``,
``solve_qp`` and ``reconstruct_states``.  ``install(ref_mpc)`` rebinds those
globals to this package's GPU functions, so the reference's own control logic
(SQP loop, damping, fallback policies, input filter, shift, MpcState) runs
unchanged on top of the sm_100a kernels; ``uninstall`` restores them.

The reference's types stay the reference's: ``solve_qp`` is wrapped so the
reference ``QpProblem`` / ``SolverSettings`` go in and a reference
``QpSolution`` carrying the reference ``QpStatus`` comes out (``mpc_step``
compares ``sol.status`` against its own enum, ``mpc.py:146``).  Everything
else is duck-typed: the reference's ``GnnModel``, ``GraphTopology``,
``OcpSpec`` and NumPy arrays are accepted by the GPU functions as they are.
"""

from __future__ import annotations

import sys

from . import condensing as _cond
from . import gnn as _gnn
from . import qpsolver as _qp

STAGES = ("linearize_trajectory", "condense_gammas", "condense_ocp", "expand_soft_constraints",
          "reconstruct_states", "solve_qp")


def _ref_qpsolver(ref_mpc):
    """The reference's qpsolver module (sibling of the given mpc module)."""
    pkg = ref_mpc.__name__.rsplit(".", 1)[0]
    return sys.modules[f"{pkg}.qpsolver"]


def solve_qp_for(ref_qpsolver):
    """A ``solve_qp`` with the reference's signature and return type that runs
    K-QP (``qpsolver.py:112-235``)."""

    def solve_qp(problem, settings=None):
        sol = _qp.solve_qp(problem, settings)
        return ref_qpsolver.QpSolution(
            u=sol.u, duals=sol.duals, status=ref_qpsolver.QpStatus(sol.status.value),
            iterations=sol.iterations, stationarity=sol.stationarity,
            primal_infeas=sol.primal_infeas, complementarity=sol.complementarity)

    solve_qp.__doc__ = _qp.solve_qp.__doc__
    return solve_qp


def install(ref_mpc) -> dict:
    """Rebind the stage functions of the reference module ``ref_mpc``
    (``gnnmpc.mpc``) to the B200 path; returns the originals (pass them to
    ``uninstall``)."""
    saved = {name: getattr(ref_mpc, name) for name in STAGES}
    ref_mpc.linearize_trajectory = _gnn.linearize_trajectory
    ref_mpc.condense_gammas = _cond.condense_gammas
    ref_mpc.condense_ocp = _cond.condense_ocp
    ref_mpc.expand_soft_constraints = _cond.expand_soft_constraints
    ref_mpc.reconstruct_states = _cond.reconstruct_states
    ref_mpc.solve_qp = solve_qp_for(_ref_qpsolver(ref_mpc))
    return saved


def uninstall(ref_mpc, saved: dict) -> None:
    for name, fn in saved.items():
        setattr(ref_mpc, name, fn)
