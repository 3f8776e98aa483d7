"""Synthetic benchmark instances -- the reference's own recipe.

``scaling_problem`` restates ``_scaling_problem`` (``gnnmpc/experiments.py:
465-489``) draw for draw (same ``default_rng`` stream, same order), so a seed
gives bit-identical model weights, states, inputs and OCP data on both sides
(pinned in ``tests/test_oracle_golden.py``).  The mesh variant (cfg5) and the
batched instances (cfg4) follow SURVEY.md section 8(d).
"""

from __future__ import annotations

import numpy as np

from .condensing import OcpSpec, StateConstraint, stage_input_box
from .gnn import init_model
from .graph import chain_topology, mesh_topology


def _ocp(topo, states0, N, M):
    q = np.zeros((M, N + 1, 6, 6))
    q[:, :] = np.diag(np.concatenate([np.full(3, 1.0), np.full(3, 0.1)]))
    x_ref = states0[:, None, :].repeat(N + 1, axis=1)
    r = np.tile(np.eye(6) * 1e-2, (N, 1, 1))
    u_ref = np.zeros((N, 6))
    cons = [stage_input_box(6, 0.0, 8.0)] * N
    row = np.zeros((1, 6))
    row[0, 2] = 1.0  # end-effector height bound, one soft row per stage
    scons = [StateConstraint(M - 1, k, row, np.array([1.0]), soft=True) for k in range(1, N + 1)]
    return OcpSpec(topo, N, q, x_ref, r, u_ref, cons, scons)


def scaling_problem(M: int, N: int, dt: float = 0.01, seed: int = 0):
    """Chain instance: returns (topo, model, states (N,M,6), inputs (N,6), spec)."""
    rng = np.random.default_rng(seed)
    topo = chain_topology(M)
    model = init_model(3, 6, dt, rng, n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64),
                       out_scale=0.05)
    states = np.zeros((N, M, 6))
    states[:, :, 2] = -0.15 * np.arange(M)
    states += 0.01 * rng.standard_normal(states.shape)
    inputs = rng.uniform(0.0, 4.0, size=(N, 6))
    return topo, model, states, inputs, _ocp(topo, states[0], N, M)


def mesh_problem(rows: int, cols: int, N: int, dt: float = 0.01, seed: int = 0):
    """2-D mesh instance (cfg5): nodes on a 0.15 m grid (x = 0.15 c,
    z = -0.15 r) plus 0.01 noise; otherwise the scaling recipe."""
    rng = np.random.default_rng(seed)
    topo = mesh_topology(rows, cols)
    M = rows * cols
    model = init_model(3, 6, dt, rng, n_m=16, psi_hidden=(32, 32), phi_hidden=(64, 64),
                       out_scale=0.05)
    ids = np.arange(M)
    states = np.zeros((N, M, 6))
    states[:, :, 0] = 0.15 * (ids % cols)
    states[:, :, 2] = -0.15 * (ids // cols)
    states += 0.01 * rng.standard_normal(states.shape)
    inputs = rng.uniform(0.0, 4.0, size=(N, 6))
    return topo, model, states, inputs, _ocp(topo, states[0], N, M)


def batch_instance(b: int, M: int, N: int):
    """Per-instance states / inputs of cfg4 instance b (rng = default_rng(1+b))."""
    rng = np.random.default_rng(1 + b)
    states = np.zeros((N, M, 6))
    states[:, :, 2] = -0.15 * np.arange(M)
    states += 0.01 * rng.standard_normal(states.shape)
    inputs = rng.uniform(0.0, 4.0, size=(N, 6))
    return states, inputs
