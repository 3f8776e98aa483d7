"""Debug: k_condense_tc vs SIMT fused on several shapes; per-block H error map."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_gpu_fused import _run
from paper_2602_17601_b200.graph import chain_topology, mesh_topology

for name, topo, N, nx, nu in [("chain37", chain_topology(37), 5, 6, 6), ("chain8", chain_topology(8), 3, 6, 6),
                              ("chain1000", chain_topology(1000), 20, 6, 6), ("chain1000n4", chain_topology(1000), 4, 6, 6),
                              ("mesh", mesh_topology(23, 17), 12, 6, 3), ("c37_2_1", chain_topology(37), 5, 2, 1)]:
    ref, outs = _run(topo, N, nx, nu, 1, seed=11, reps=1, mode=0)
    W1, H1, g1 = ref
    W2, H2, g2 = outs[0]
    Hr, Hf = H1.cpu().numpy()[0], H2.cpu().numpy()[0]
    gr, gf = g1.cpu().numpy()[0], g2.cpu().numpy()[0]
    scale = np.max(np.abs(Hr))
    eH = np.abs(Hf - Hr) / scale
    print(f"{name}: N={N} nu={nu} H err {eH.max():.3e} g err {np.max(np.abs(gf-gr))/max(1,np.max(np.abs(gr))):.3e} "
          f"nan={np.isnan(Hf).sum()}")
    if eH.max() > 1e-5:
        blk = eH.reshape(N, nu, N, nu).max(axis=(1, 3))
        np.set_printoptions(linewidth=250, precision=1)
        print(np.log10(blk + 1e-30).round(0))
        i, j = np.unravel_index(np.argmax(eH), eH.shape)
        print("worst", i, j, Hf[i, j], Hr[i, j])
        print("diag ratio", (np.diag(Hf) / np.diag(Hr))[:24])
