"""B200-native GNN-MPC hot path (arXiv 2602.17601): linearize -> condense ->
H/g reduction -> QP, as hand-written sm_100a kernels behind a C ABI
(``include/gnnmpc_b200.h``), exposed through the reference package's Python
API so it is a drop-in for ``gnnmpc``'s per-step path.

Pure-data modules (graph, mlp, model types, OCP types) import without a GPU;
every computing entry point needs the native library and a CUDA device and
raises otherwise -- there is no CPU fallback.
"""

from .errors import ConfigurationError
from .graph import (GraphTopology, InputVector, NodeState, SystemState, Trajectory,
                    chain_topology, flatten_state, mesh_topology, unflatten_state)
from .gnn import (GnnModel, LinearizedDynamics, Normalization, gnn_step, init_model,
                  linearize_stage, linearize_trajectory, load_model, rollout, save_model,
                  step_array)
from .mlp import MlpParams, mlp_init
from .qpsolver import QpProblem, QpSolution, QpStatus, SolverSettings, solve_qp, solve_qp_batched
from .condensing import (CondensedQp, LocalCondensed, OcpSpec, StateConstraint, assemble_qp,
                         condense_gammas, condense_local, condense_ocp, cost_to_standard_form,
                         expand_soft_constraints, local_hessian_gradient, reconstruct_states,
                         stage_input_box)
from .mpc import (ClosedLoopLog, MpcConfig, MpcState, StepTiming, mpc_init, mpc_step,
                  run_closed_loop)

__version__ = "0.1.0"
