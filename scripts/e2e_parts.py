"""Host-side costs of the pieces of mpc_step at cfg3 (diagnostics)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2602_17601_b200 as pkg
from paper_2602_17601_b200 import workloads, mpc as M, device as D

topo, model, states, inputs, spec = workloads.scaling_problem(1000, 20, 0.01, 0)
spec.freeze(); model.freeze()
cfg = pkg.MpcConfig(horizon=20, dt=0.01)
dev = torch.device("cuda", 0)
state = pkg.MpcState(lin_states=torch.from_numpy(np.tile(states[0], (21, 1, 1))).to(dev),
                     lin_inputs=torch.zeros((20, 6), dtype=torch.float64, device=dev))
xs = pkg.SystemState(states[0])
for _ in range(10):
    u, state = pkg.mpc_step(model, topo, spec, xs, state, cfg)
torch.cuda.synchronize()
eng = D.engine(topo, model)
plan = M.get_plan(eng, spec, 20, 6, 6, cfg, True)

def t(fn, n=2000):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6

print("engine()          us", t(lambda: D.engine(topo, model)))
print("get_plan          us", t(lambda: M.get_plan(eng, spec, 20, 6, 6, cfg, True)))
print("host_x fill       us", t(lambda: plan.host_x.numpy().__setitem__(Ellipsis, np.asarray(xs.array, dtype=float).reshape(plan.host_x.shape))))
ls_src = state.device_value("lin_states")
print("ls copy_ (D2D)    us", t(lambda: plan.ls.copy_(ls_src)))
print("u_prev zero_      us", t(lambda: plan.u_prev.zero_()))
print("stage_ms          us", t(lambda: plan.stage_ms()))
print("outbuf clone      us", t(lambda: plan.outbuf.clone()))
print("u_applied clone   us", t(lambda: plan.u_applied.clone()))
print("carve             us", t(lambda: plan._carve(plan.outbuf)))
print("MpcState()        us", t(lambda: M.MpcState(lin_states=ls_src, lin_inputs=ls_src)))
print("InputVector       us", t(lambda: pkg.InputVector(np.zeros(6))))
print("stream sync idle  us", t(lambda: torch.cuda.current_stream(dev).synchronize()))
print("mpc_step total    us", t(lambda: pkg.mpc_step(model, topo, spec, xs, state, cfg), n=300))
print("graph replay+sync us", t(lambda: (plan.graph.replay(), torch.cuda.current_stream(dev).synchronize()), n=300))
ev = plan.events
print("torch elapsed     ", ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]))
print("gm_event_times    ", plan.stage_ms())
