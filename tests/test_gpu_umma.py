"""Known-answer test of the tcgen05 3xTF32 Gram product (csrc/umma.cuh) that
K-COND uses for the node reduction of H (condensing.py:383-389):
S = G' Q accumulated in TMEM over K rows streamed through shared memory.

Tolerance: 3xTF32 with fp32 accumulation is ~fp32 accurate; against an fp64
product the bound is max|S - S_ref| <= 1e-5 * sum_k |G| |Q| (elementwise), far
below the 1e-4 relative bound on H.  Plain TF32 would
miss it by ~100x, which is what the test guards against."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,P", [(8, 6), (48, 16), (96, 120), (130, 120), (1000, 120), (37, 33), (480, 128)])
def test_gram_3xtf32(K, P):
    import torch

    from paper_2602_17601_b200 import chain_topology, device

    rng = np.random.default_rng(K * 1000 + P)
    G = rng.standard_normal((K, P)).astype(np.float32)
    Q = rng.standard_normal((K, P)).astype(np.float32)
    eng = device.engine(chain_topology(1))
    dG, dQ = eng.h2d(G, np.float32), eng.h2d(Q, np.float32)
    S = eng.empty((P, P), np.float32)
    eng.ctx.call("gm_gram_check", K, P, dG.data_ptr(), dQ.data_ptr(), S.data_ptr(), eng.stream_ptr())
    torch.cuda.synchronize()
    ref = G.astype(np.float64).T @ Q.astype(np.float64)
    scale = np.abs(G.astype(np.float64)).T @ np.abs(Q.astype(np.float64))
    err = np.abs(S.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * scale + 1e-30), float(np.max(err / scale))
