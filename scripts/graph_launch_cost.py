"""CPU cost of launching the cfg3 step graph (diagnostics): replay() of the
whole-step graph, and variants captured without timing events / copies."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads, mpc as M

topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze(); model.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
xs = pkg.SystemState(states[0])
dev = torch.device("cuda", 0)
st0 = pkg.MpcState(lin_states=torch.from_numpy(np.tile(states[0], (21, 1, 1))).to(dev),
                   lin_inputs=torch.zeros((20, 6), dtype=torch.float64, device=dev))
for _ in range(5):
    pkg.mpc_step(model, topo, spec, xs, st0, cfg)
torch.cuda.synchronize()

from paper_2602_17601_b200.device import engine
eng = engine(topo, model)
plans = [v for k, v in eng.cache.items() if isinstance(v, M.StepPlan)] if hasattr(eng, "cache") else []
print("plans", len(plans))
plan = plans[0]
g = plan.graph

def t_replay(graph, n=200):
    torch.cuda.synchronize()
    cpu = 0.0
    for _ in range(n):
        t0 = time.perf_counter(); graph.replay(); cpu += time.perf_counter() - t0
        torch.cuda.synchronize()
    return cpu / n * 1e6

print("whole-step graph replay CPU us", t_replay(g))
for i, gg in enumerate(plan.graphs):
    print(f"group graph {i} replay CPU us", t_replay(gg))
# variant: groups captured in one graph without events / copies
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    plan._issue(plan.groups(), eager=True, timed=False)
print("one graph, no events/copies, CPU us", t_replay(g2))
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3):
    plan._issue(plan.groups(), eager=True, timed=True)
print("one graph, events, no copies, CPU us", t_replay(g3))
# end-to-end wall per replay incl. sync
for name, gg in (("whole", g), ("noev", g2)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(200):
        gg.replay(); torch.cuda.synchronize()
    print(name, "replay+sync ms", (time.perf_counter() - t0) / 200 * 1e3)
