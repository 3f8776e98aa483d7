"""MLP parameter container and initialisation (host side, pure data).

``MlpParams`` / ``mlp_init`` mirror ``gnnmpc/mlp.py:15-78``: weights[l] has
shape ``(layer_dims[l+1], layer_dims[l])`` (row-major, out x in), ReLU on
hidden layers, affine output.  ``mlp_init`` draws from the caller's
``numpy.random.Generator`` in the same order and with the same arithmetic
as the reference, so a seed produces bit-identical weights on both sides
(pinned by ``tests/test_oracle_golden.py``).

The forward pass and input Jacobian themselves run on the GPU inside the
fused linearisation kernel (``csrc/k_linearize.cu``); nothing here computes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class MlpParams:
    layer_dims: list
    weights: list
    biases: list

    def __post_init__(self):
        dims = [int(d) for d in self.layer_dims]
        if len(dims) < 2 or any(d < 1 for d in dims):
            raise ValueError("layer_dims needs >= 2 positive entries")
        if len(self.weights) != len(dims) - 1 or len(self.biases) != len(dims) - 1:
            raise ValueError("need one weight/bias pair per layer")
        self.weights = list(self.weights)
        self.biases = list(self.biases)
        for l in range(len(dims) - 1):
            W = np.asarray(self.weights[l], dtype=float)
            b = np.asarray(self.biases[l], dtype=float)
            if W.shape != (dims[l + 1], dims[l]) or b.shape != (dims[l + 1],):
                raise ValueError(f"layer {l} shape mismatch with layer_dims")
            if not (np.all(np.isfinite(W)) and np.all(np.isfinite(b))):
                raise ValueError("parameters must be finite")
            self.weights[l] = W
            self.biases[l] = b
        self.layer_dims = dims

    @property
    def in_dim(self) -> int:
        return self.layer_dims[0]

    @property
    def out_dim(self) -> int:
        return self.layer_dims[-1]

    @property
    def n_layers(self) -> int:
        return len(self.weights)

    def copy(self) -> "MlpParams":
        return MlpParams(list(self.layer_dims), [W.copy() for W in self.weights],
                         [b.copy() for b in self.biases])

    def param_sq_norm(self) -> float:
        return float(sum(np.sum(W * W) for W in self.weights)
                     + sum(np.sum(b * b) for b in self.biases))


def mlp_init(layer_dims, rng: np.random.Generator, out_scale: float = 1.0) -> MlpParams:
    """He-normal weights, zero biases, ``out_scale`` on the output layer
    (draw order and arithmetic as ``gnnmpc/mlp.py:67-78``)."""
    dims = [int(d) for d in layer_dims]
    weights, biases = [], []
    last = len(dims) - 2
    for l in range(len(dims) - 1):
        fan_in = dims[l]
        W = rng.standard_normal((dims[l + 1], fan_in)) * np.sqrt(2.0 / fan_in)
        if l == last:
            W *= out_scale
        weights.append(W)
        biases.append(np.zeros(dims[l + 1]))
    return MlpParams(dims, weights, biases)
