"""Benchmark of the B200 GNN-MPC hot path (one RTI step: linearize + condense +
QP + epilogue) on BASELINE.json's headline workload, cfg3: chain graph with
M = 1,000 nodes, horizon N = 20 (the paper's 100 Hz claim).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on stdout (rank 0).  A "step" is one mpc_step of the cfg3
instance from the same initial controller state (identical work every step):

* value      device time of the captured kernel chain with every input already
             in HBM, L2 flushed (256 MiB write) between timed steps; whole-job
             solves/s = n_gpus * 1000 / max-over-ranks ms.
* e2e        the public API mpc_step(model, topo, spec, x_measured, state, cfg)
             with the measurement in pinned host memory: H2D of x_measured,
             the kernels, D2H of [u_applied, status, iterations], wall clock.
* roofline   the dominant kernel (per-launch CUDA-event time inside the timed
             region) against its hardware ceiling.
* cpu_baseline / --impl reference: the reference's own CPU path -- the
  unmodified package installed in baseline/_ref (pip --target), called
  through its public mpc_step; the oracle port (oracle/ref_port.py) only when
  that install is missing.

Multi-GPU (torchrun): every rank solves its own independent instance (weak
scaling, no data-path collective); timing is max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPC step latency ms (linearize+condense+QP) & Hz at N nodes; solves/sec batched"
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the round's
# `ncu --set full` captures at cfg3 (profiles/r01/ncu_full_summary_v8.txt)
NCU_TRAFFIC = {"k_solve_qp": 757760, "linearize": None, "k_condense_tc": 38191616}
# sm__pipe_tensor_cycles_active (% of peak, active cycles) of K-COND's tcgen05
# H/g accumulation from the same capture
NCU_TENSOR_PCT = {"k_condense_tc": 4.62,
                  # cfg3 (v8 / v7 captures): fp64 DMMA forward chain, tcgen05 Jacobians
                  "linearize": {"k_fwd_chain_mma<phi>": 30.5, "k_jac_phi_tc": 8.4, "k_jac_psi_tc": 6.3}}
# cfg3 linearize flops, psi-VJP formulation
LIN_FLOPS_CFG3 = 1.53e9
M_NODES, HORIZON = 1000, 20
WORKLOAD = "cfg3: chain graph M=1000 nodes, horizon N=20, _scaling_problem recipe (paper 100 Hz headline)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--nodes", type=int, default=M_NODES)
    ap.add_argument("--horizon", type=int, default=HORIZON)
    ap.add_argument("--cpu-steps", type=int, default=8, help="oracle steps for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-l2-flush", action="store_true")
    ap.add_argument("--workload", choices=["cfg2", "cfg3", "cfg4", "cfg5"], default="cfg3",
                    help="cfg3 (default, headline latency); cfg4: 4096 instances of M=200 "
                         "sharded over ranks; cfg5: 400x250 mesh, node-partitioned over ranks")
    ap.add_argument("--batch", type=int, default=4096, help="cfg4 total instances")
    ap.add_argument("--wave", type=int, default=1024, help="cfg4 instances per launch wave")
    return ap.parse_args()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def problem(M, N):
    from paper_2602_17601_b200 import workloads

    topo, model, states, inputs, spec = workloads.scaling_problem(M, N, 0.01, 0)
    return topo, model, states, inputs, spec


# ---------------------------------------------------------------------------
# CPU legs (oracle port = the reference algorithm on the host cores)
# ---------------------------------------------------------------------------

def cpu_oracle_steps(M, N, steps, warmup, threads):
    from threadpoolctl import threadpool_limits

    from oracle import ref_port as O

    topo, model, states, inputs, spec = problem(M, N)
    x0 = states[0]
    ls0 = np.tile(x0, (N + 1, 1, 1))
    li0 = np.zeros((N, 6))
    times = []
    with threadpool_limits(limits=threads):
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            O.mpc_step(model, topo, spec, x0, ls0, li0, N, threads=threads)
            dt = time.perf_counter() - t0
            if k >= warmup:
                times.append(dt)
    return float(np.mean(times)) * 1e3


def import_reference():
    """The unmodified reference package installed in baseline/_ref (pip
    --target), or None when it is not there."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "gnnmpc" / "mpc.py").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import gnnmpc.experiments as rex
        import gnnmpc.graph as rgr
        import gnnmpc.mpc as rm
    finally:
        sys.path.remove(str(ref))
    return rex, rgr, rm


def reference_steps(M, N, steps, warmup, threads):
    """Stock reference mpc_step (gnnmpc.mpc, mpc.py:102-200) on the
    reference's own _scaling_problem (experiments.py:465-489), from the same
    initial controller state every step (the work of our arm's step).
    Returns (ms per step, status, iterations)."""
    from threadpoolctl import threadpool_limits

    rex, rgr, rm = import_reference()
    topo, model, states, inputs, spec = rex._scaling_problem(M, N, 0.01, 0)
    cfg = rm.MpcConfig(horizon=N, dt=0.01, threads=threads)
    x = rgr.SystemState(states[0])
    st0 = rm.mpc_init(x, cfg, 6)
    times = []
    with threadpool_limits(limits=threads):
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            u, st1 = rm.mpc_step(model, topo, spec, x, st0, cfg)
            dt = time.perf_counter() - t0
            if k >= warmup:
                times.append(dt)
    return float(np.mean(times)) * 1e3, st1.last_status.value, st1.last_iterations


def reference_arm(args, world, rank):
    """The reference's own CPU implementation of the path, timed on the host
    cores: the unmodified package from baseline/_ref through its public
    mpc_step (BLAS threads = condense threads = all cores); the oracle port
    only if the install is missing.  Rank 0 alone runs at N>1."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    M, N = args.nodes, args.horizon
    if import_reference() is not None:
        ms, status, iters = reference_steps(M, N, args.steps, args.warmup, cores)
        kind = "reference"
        what = (f"{args.steps} calls of the unmodified reference gnnmpc.mpc.mpc_step "
                f"(baseline/_ref) after {args.warmup} warm-up, M={M}, N={N}, "
                f"_scaling_problem seed 0, BLAS threads = condense threads = {cores}")
    else:
        ms = cpu_oracle_steps(M, N, args.steps, args.warmup, cores)
        status, iters = None, None
        kind = "port"
        what = (f"{args.steps} oracle mpc_step calls (after {args.warmup} warm-up) at M={M}, "
                f"N={N}, BLAS threads = condense threads = {cores} (baseline/_ref missing)")
    v = 1000.0 / ms
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "nodes": M, "horizon": N,
                                        "parallelism": "host cores",
                                        "qp": {"status": status, "iterations": iters}},
        "cpu_baseline": {"value": v, "unit": "solves/s", "cores": cores, "kind": kind,
                         "sample": what},
        "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self, wait_s=5.0):
        """Start sampling every 50 ms; returns once the first sample arrived
        (nvidia-smi can take a second to come up) so the timed region that
        follows is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        t0 = time.time()
        while not self.lines and time.time() - t0 < wait_s:
            time.sleep(0.02)
        self.n0 = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                smax = float(parts[2].split()[0])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def qp_flops(n, m, ng, iters):
    """Algorithmic fp64 flops of the IPM on the expanded QP (qpsolver.py:170-229):
    per iteration Schur build 2*ng*n^2/2, Cholesky n^3/3, 4 triangular solves 4n^2,
    H u / C products ~ 2n^2 + 4 m n (dense count of single-nonzero rows excluded)."""
    per = ng * n * n + n ** 3 / 3.0 + 4.0 * n * n + 2.0 * n * n + 4.0 * ng * n
    return per * max(iters, 1)


def ours_arm(args, world, rank, local):
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime
    from paper_2602_17601_b200.mpc import get_plan

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    M, N = args.nodes, args.horizon
    topo, model, states, inputs, spec = problem(M, N)
    spec.freeze()
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x0 = states[0]
    xs = pkg.SystemState(x0)
    # device-resident initial controller state (mpc_init values)
    st0 = pkg.MpcState(lin_states=torch.from_numpy(np.tile(x0, (N + 1, 1, 1))).to(dev),
                       lin_inputs=torch.zeros((N, 6), dtype=torch.float64, device=dev))
    # first calls: upload, eager run, CUDA-graph capture
    for _ in range(3):
        u, st1 = pkg.mpc_step(model, topo, spec, xs, st0, cfg)
    eng = pkg.device.engine(topo, model)
    plan = get_plan(eng, spec, N, 6, 6, cfg, True)
    assert plan.graphs is not None, "plan was not captured as CUDA graphs"
    status, iters = st1.last_status.value, st1.last_iterations

    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    L = _runtime.lib()

    # ---- device-resident timing (value) ----
    for _ in range(args.warmup):
        plan.enqueue(timed=True)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms, lin_ms, cond_ms, solve_ms = [], [], [], []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        if not args.no_l2_flush:
            flush.fill_(1.0)
        plan.enqueue(timed=True)
        torch.cuda.synchronize()
        a, b, c = plan.stage_ms()
        lin_ms.append(a)
        cond_ms.append(b)
        solve_ms.append(c)
        step_ms.append(plan.events[0].elapsed_time(plan.events[3]))
    torch.cuda.synchronize()
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # ---- end to end through the public API (value e2e) ----
    e2e = []
    for _ in range(args.warmup):
        pkg.mpc_step(model, topo, spec, xs, st0, cfg)
    for _ in range(args.steps):
        if not args.no_l2_flush:
            flush.fill_(1.0)
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, st1 = pkg.mpc_step(model, topo, spec, xs, st0, cfg)
        e2e.append(time.perf_counter() - t0)
    clk = clocks.stop()
    e2e_ms = float(np.mean(e2e)) * 1e3
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # kernels launched per step: count one eager (uncaptured) enqueue
    l1 = L.gm_launch_count()
    saved = plan.graphs
    plan.graphs = None
    plan.enqueue(timed=False)
    plan.graphs = saved
    torch.cuda.synchronize()
    kernels_per_step = int(L.gm_launch_count() - l1)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    # ---- roofline of the dominant kernel ----
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_path.read_text()) if peaks_path.exists() else {}
    smax = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    solve = float(np.mean(solve_ms))
    n, m = plan.n, plan.m
    ng = plan.ds.ns + (plan.ds.rows.n_st)  # general (multi-nonzero) rows: the soft rows
    fl = qp_flops(n, m, ng, iters)
    fp64_sm_peak = 64 * 2 * smax / 1e12  # one CTA on one SM: 64 DFMA/clk
    roof = {"kernel": "k_solve_qp (+k_finish)", "bound": "tensor",
            "achieved": fl / (solve * 1e-3) / 1e12, "peak": fp64_sm_peak, "unit": "TFLOP/s",
            "frac": (fl / (solve * 1e-3) / 1e12) / fp64_sm_peak, "traffic": None,
            "note": "single-CTA fp64 IPM (Schur build and Cholesky updates on fp64 DMMA); peak = the fp64 "
                    "tensor/FMA rate of the ONE SM it runs on at max clock (64 DFMA/clk); latency-bound"}

    # HBM roofline of the Gamma recursion + H/g kernel (K-COND): compulsory
    # bytes of the recursion (read stage n of Gamma once, write
    # stage n+1 once, causal columns only, fp32) plus the A/B/c blocks
    nx, nu = 6, 6
    gam = 4.0 * M * nx * sum((1 + k * nu) + (1 + (k + 1) * nu) for k in range(N))
    blocks = N * (M * nx * nx * 4 + int(topo.edge_count) * nx * nx * 4
                  + M * nx * nu * 4 + M * nx * 8)
    cond = float(np.mean(cond_ms))
    hbm_peak = float(peaks.get("hbm_gbs") or 6449.1)
    cond_gbs = (gam + blocks) / (cond * 1e-3) / 1e9
    # H on the tensor cores: causal Gram flops x3 (3xTF32) against
    # the dense tf32 peak
    hfl = M * sum(2 * nx * nx * k * nu + 2 * nx * (k * nu) ** 2 for k in range(1, N + 1))
    tf32_peak = float(peaks.get("tf32_tflops") or 1100.0)
    # K-LIN: algorithmic flops of the psi-VJP formulation, FP32 SIMT
    lin = float(np.mean(lin_ms))
    stages = {
        "k_condense_tc": {"bound": "hbm", "achieved": cond_gbs, "peak": hbm_peak, "unit": "GB/s",
                          "frac": cond_gbs / hbm_peak, "algorithmic_bytes": gam + blocks,
                          "traffic": NCU_TRAFFIC.get("k_condense_tc"),
                          "h_tensor": {"algorithmic_flops": hfl, "issued_tf32_flops": 3 * hfl,
                                       "achieved_tflops": 3 * hfl / (cond * 1e-3) / 1e12,
                                       "peak_tflops": tf32_peak,
                                       "tensor_pipe_pct_ncu": NCU_TENSOR_PCT.get("k_condense_tc")},
                          "note": "stage time incl. constraint rows/soft expansion; Gamma is L2-resident at cfg3; "
                                  "H and g accumulate on tcgen05 (3xTF32) inside the recursion kernel"},
        "linearize": {"bound": "tensor (fp64 DMMA forward, tcgen05 3xTF32 Jacobians)", "ms": lin,
                      "kernels": "k_fwd_chain_mma (psi, phi; fp64 DMMA), k_jac_phi_tc, k_jac_psi_tc (tcgen05 "
                                 "3xTF32), k_lin_self, k_lin_c, k_lin_f",
                      "achieved": LIN_FLOPS_CFG3 / (lin * 1e-3) / 1e12 if (M, N) == (1000, 20) else None,
                      "unit": "TFLOP/s", "traffic": NCU_TRAFFIC.get("linearize"),
                      "tensor_pipe_pct_ncu": NCU_TENSOR_PCT.get("linearize"),
                      "note": "stage of 6 short launches (~0.12 ms at cfg3): launch/tail-bound; tensor pipe "
                              "activity per kernel from ncu in tensor_pipe_pct_ncu"},
    }
    roof["traffic"] = NCU_TRAFFIC.get("k_solve_qp")

    cpu = None
    if not args.no_cpu_baseline:
        if import_reference() is not None:
            cms = reference_steps(M, N, args.cpu_steps, 1, 1)[0]
            kind, who = "reference", "unmodified reference gnnmpc.mpc.mpc_step (baseline/_ref)"
        else:
            cms = cpu_oracle_steps(M, N, args.cpu_steps, 1, 1)
            kind, who = "port", "oracle mpc_step (baseline/_ref missing)"
        cpu = {"value": 1000.0 / cms, "unit": "solves/s", "cores": 1, "kind": kind,
               "sample": f"{args.cpu_steps} calls of the {who} at M={M}, N={N} (1 warm-up), "
                         "BLAS pinned to 1 thread (reference protocol experiments.py:492-528)",
               "ms_per_step": cms}
    out = {
        "metric": METRIC, "value": world * 1000.0 / ms, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "hz": 1000.0 / ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (linearize Jacobians, Gamma, H) / f64 (MLP forward, offsets, QP)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": M, "horizon": N, "instances_per_gpu": 1,
                   "parallelism": f"independent instance per GPU x{world}",
                   "l2": "flushed (256 MiB write) between timed steps" if not args.no_l2_flush
                   else "not flushed", "qp": {"n": n, "m": m, "status": status,
                                              "iterations": iters}},
        "stage_ms": {"linearize": float(np.mean(lin_ms)), "condense": float(np.mean(cond_ms)),
                     "solve_and_epilogue": solve},
        "e2e": {"value": world * 1000.0 / e2e_ms, "unit": "solves/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": M * 6 * 8, "d2h_bytes_per_step": (6 + 2) * 8,
                "path": "paper_2602_17601_b200.mpc_step (public API), host numpy measurement"},
        "gpu_launches": kernels_per_step,
        "gpu_launch_mode": "CUDA graphs (3 replays/step)",
        "clocks": clk,
        "roofline": roof,
        "roofline_stages": stages,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cfg4_arm(args, world, rank, local):
    """4096 independent M=200, N=20 instances, sharded over ranks (strong
    scaling of a fixed batch; no data-path collective).  value: device time
    of all waves with every input resident in HBM (one device-to-device load
    per wave into the batch buffers + the kernel chain); e2e: batch.WavePipeline
    from pinned host arrays (H2D of each wave's inputs on a side stream under
    the previous wave's kernels, D2H of u/status)."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.batch import BatchedMpc, WavePipeline, shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    M, N = 200, 20
    topo, model, _, _, spec = workloads.scaling_problem(M, N, 0.01, 0)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    lo, hi = shard_range(args.batch, world, rank)
    waves = [(a, min(a + args.wave, hi)) for a in range(lo, hi, args.wave)]
    host, resident = [], []
    for a, b in waves:
        xs, ls, li, xr = [], [], [], []
        for i in range(a, b):
            st, inp = workloads.batch_instance(i, M, N)
            xs.append(st[0]); ls.append(np.concatenate([st, st[-1:]], 0)); li.append(inp)
            xr.append(np.repeat(st[0][:, None, :], N + 1, axis=1))
        arrs = [torch.from_numpy(np.stack(v)).pin_memory() for v in (xs, ls, li, xr)]
        host.append(arrs)
        resident.append([t.to(dev) for t in arrs])
    bms = {}
    def bm_for(n):
        if n not in bms:
            bms[n] = BatchedMpc(model, topo, spec, cfg, n)
        return bms[n]
    def device_step():
        for (a, b), d in zip(waves, resident):
            bm = bm_for(b - a)
            bm.load(*d)
            bm.enqueue()
    # e2e: the public WavePipeline (each wave's H2D on a side stream under the
    # previous wave's kernels, one host sync per step)
    pipe = WavePipeline(model, topo, spec, cfg, [b - a for a, b in waves])
    def e2e_step():
        return pipe.step(host)
    for _ in range(args.warmup):
        device_step()
        e2e_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local); clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(args.steps):
        ev0.record()
        device_step()
        ev1.record()
        torch.cuda.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    dev_ms = float(np.mean(ms))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = e2e_step()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) / args.steps * 1e3
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([dev_ms, e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, e2e_ms = (float(v) for v in t.tolist())
    if rank == 0:
        iters = [int(i) for r in res for i in r.iterations]
        per = hi - lo
        print(json.dumps({
            "metric": METRIC, "value": args.batch / (dev_ms * 1e-3), "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": f"cfg4: {args.batch} independent chain M=200, N=20 instances",
                       "instances_per_gpu": per, "wave": args.wave,
                       "parallelism": f"instance shards x{world}",
                       "qp_iterations_mean_rank0": float(np.mean(iters))},
            "e2e": {"value": args.batch / (e2e_ms * 1e-3), "unit": "solves/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": per * (M * 6 + (N + 1) * M * 6 + N * 6 + M * (N + 1) * 6) * 8,
                    "d2h_bytes_per_step": per * 8 * 8,
                    "path": "batch.WavePipeline.step from pinned host arrays (H2D overlapped with the previous wave's kernels; wall clock)"},
            "clocks": clk}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cfg2_arm(args, world, rank, local):
    """Closed-loop tracking, chain M=100 (BASELINE cfg2): ChainConfig(100),
    settled 3 s, end effector on a 0.04 m / 8 s circle around its settled
    position, default TrackingWeights, random-init GNN (no training data),
    horizon 20.  A step = one controller step (mpc_step) + one plant period
    (device kernel); the state stays on the device, per step x_ref (H2D) and
    [u, status, iterations] (D2H) cross.  Replicas at N>1 (no collective)."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200.graph import chain_topology
    from paper_2602_17601_b200.tracking import (TrackingWeights, circle_reference,
                                                 run_closed_loop_device, tracking_spec_provider)
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    M, N = 100, 20
    pc = ChainConfig(node_count=M)
    topo = chain_topology(M)
    model = pkg.init_model(3, 6, 0.01, np.random.default_rng(0), out_scale=0.05)
    plant = DevicePlant(pc, topo)
    x0 = plant.settle(3.0)
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    center = x0[-1, :3].cpu().numpy()
    prov = tracking_spec_provider(topo, cfg, pkg.SystemState(x0.cpu().numpy()),
                                  circle_reference(0.04, 8.0, center), TrackingWeights(), pc.n_u, pc.u_max)
    run_closed_loop_device(plant, model, topo, prov, x0, args.warmup, cfg)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local); clocks.start()
    t0 = time.perf_counter()
    log = run_closed_loop_device(plant, model, topo, prov, x0, args.steps, cfg)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / args.steps * 1e3
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    tm = log.timings.mean(axis=0)
    cpu = None
    if not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits

        from oracle import ref_port as O
        P = O.trunk_params(M)
        specs = O.tracking_specs(topo, N, 0.01, x0.cpu().numpy(), O.circle_ref(0.04, 8.0, center), 6, 8.0)
        n_cpu = max(2, min(args.cpu_steps, 6))
        with threadpool_limits(limits=1):
            c0 = time.perf_counter()
            O.closed_loop(model, topo, P, specs, x0.cpu().numpy(), n_cpu, N)
            cms = (time.perf_counter() - c0) / n_cpu * 1e3
        cpu = {"value": 1000.0 / cms, "unit": "steps/s", "cores": 1, "kind": "port",
               "sample": f"{n_cpu} closed-loop steps (oracle mpc_step + numpy plant) at M={M}, N={N}, "
                         "BLAS pinned to 1 thread", "ms_per_step": cms}
    print(json.dumps({
        "metric": METRIC, "value": world * 1000.0 / ms, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "hz": 1000.0 / ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (random-init GNN, trunk plant)",
        "config": {"workload": "cfg2: closed-loop tracking, soft-trunk-like chain M=100, horizon 20",
                   "plant": "trunk.py chain on the device (10 substeps)", "reference": "circle r=0.04 m, T=8 s",
                   "parallelism": f"independent closed loop per GPU x{world}",
                   "optimal_fraction": log.optimal_fraction(),
                   "mean_qp_iterations": float(np.mean(log.iterations))},
        "stage_ms": {"linearize": float(tm[0]), "condense": float(tm[1]), "solve_and_epilogue": float(tm[2]),
                     "mpc_step_total": float(tm[3])},
        "e2e": {"value": world * 1000.0 / ms, "unit": "steps/s", "ms_per_step": ms,
                "h2d_bytes_per_step": M * (N + 1) * 6 * 8, "d2h_bytes_per_step": (6 + 2) * 8,
                "path": "tracking.run_closed_loop_device (public API, wall clock)"},
        "clocks": clk, "cpu_baseline": cpu}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cfg5_arm(args, world, rank, local):
    """400x250 mesh (1e5 nodes), N=20, node-partitioned over ranks with a
    per-stage NCCL halo exchange and an all-reduce of H and g."""
    import torch
    import torch.distributed as dist

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import workloads
    from paper_2602_17601_b200.partition import PartitionedMpc, partition_nodes

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    N = 20
    topo, model, states, inputs, spec = workloads.mesh_problem(400, 250, N, 0.01, 0)
    spec.freeze()
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    part = partition_nodes(topo, world, rank)
    pm = PartitionedMpc(model, topo, spec, cfg, part)
    loc = part.local_nodes  # owned + halo nodes of this rank
    ls = torch.from_numpy(np.concatenate([states, states[-1:]], 0)[:, loc]).to(dev)
    li = torch.from_numpy(inputs).to(dev)
    x0 = torch.from_numpy(states[0][loc]).to(dev)
    for _ in range(args.warmup):
        pm.step(x0, ls, li)
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local); clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(args.steps):
        ev0.record()
        u, st, it = pm.step(x0, ls, li)
        ev1.record()
        torch.cuda.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    clk = clocks.stop()
    m = torch.tensor([float(np.mean(ms))], device=dev, dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    m = float(m.item())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": 1000.0 / m, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": "cfg5: 2D mesh 400x250 = 100000 nodes, horizon 20",
                       "parallelism": (f"node partition x{world} (row slabs), NCCL halo per stage"
                                       if world > 1 else "single GPU, fused persistent recursion + cost"),
                       "qp": {"status": st, "iterations": it}},
            "e2e": {"value": 1000.0 / m, "unit": "solves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 64,
                    "path": "PartitionedMpc.step (device-resident trajectory)"},
            "clocks": clk}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    if args.workload == "cfg2":
        cfg2_arm(args, world, rank, local)
    elif args.workload == "cfg4":
        cfg4_arm(args, world, rank, local)
    elif args.workload == "cfg5":
        cfg5_arm(args, world, rank, local)
    else:
        ours_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
