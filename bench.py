"""Benchmark of the B200 GNN-MPC hot path (one RTI step: linearize + condense +
QP + epilogue) on BASELINE.json's headline workload, cfg3: chain graph with
M = 1,000 nodes, horizon N = 20 (the paper's 100 Hz claim).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg3|cfg4|cfg5|sweep] [--no-legs]

One JSON line on stdout (rank 0).  A "step" of the default workload is one
mpc_step of the cfg3 instance from the same initial controller state
(identical work every step):

* value      device time of the captured kernel chain with every input already
             in HBM, L2 flushed (256 MiB write) between timed steps; whole-job
             solves/s = n_gpus * 1000 / max-over-ranks ms (replicas).
* e2e        the public API mpc_step(model, topo, spec, x_measured, state, cfg)
             with the measurement in pinned host memory: H2D of x_measured,
             the kernels, D2H of [u_applied, status, iterations], wall clock.
* roofline   the dominant kernel (per-launch CUDA-event time inside the timed
             region, on the launching stream) against its hardware ceiling.
* legs       the sharded north_star configurations measured in the same run
             (skip with --no-legs): cfg4 (4096 x M=200 instances sharded over
             the ranks, no collective, strong scaling) and cfg5 (400x250 mesh
             node-partitioned over the ranks, NCCL halo per stage + one
             all-reduce, strong scaling), each with its own value, e2e,
             roofline, stage times and clocks.
* cpu_baseline / --impl reference: the reference's own CPU path -- the
  unmodified package installed in baseline/_ref (pip --target), called
  through its public API; the oracle port (oracle/ref_port.py) only when
  that install is missing.
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
# dram__bytes_read.sum + dram__bytes_write.sum per launch, from this round's
# `ncu --set full` captures (profiles/r02/ncu_*); None where not captured
NCU_TRAFFIC = {
    # cfg3: profiles/r02/ncu_final_kernels_v18.txt (linearize = the 6 K-LIN
    # launches of one step; K-COND = k_condense_tmap, the warp-specialised
    # TMA pipeline; k_solve_qp with the substitution solves)
    "cfg3": {"k_solve_qp": 661248, "linearize": 42505472, "k_condense": 31912448},
    # cfg4: one 1024-instance wave of k_condense_tmap (512 threads)
    "cfg4": {"k_condense": 28780996000},
    # cfg5: k_condense_tmap (512 threads, H accumulator in the global partial)
    "cfg5": {"k_condense": 27824988000},
}
M_NODES, HORIZON = 1000, 20
WORKLOAD = "cfg3: chain graph M=1000 nodes, horizon N=20, _scaling_problem recipe (paper 100 Hz headline)"
# fp64 peak: no measured figure in MEASURED_PEAKS.json; nominal B200 fp64 is
# 37 TFLOP/s = 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz
FP64_DFMA_PER_SM_CLK = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--nodes", type=int, default=M_NODES)
    ap.add_argument("--horizon", type=int, default=HORIZON)
    ap.add_argument("--cpu-steps", type=int, default=8, help="reference steps for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-l2-flush", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the cfg4 / cfg5 legs")
    ap.add_argument("--workload", choices=["cfg2", "cfg3", "cfg4", "cfg5", "sweep"], default="cfg3",
                    help="cfg3 (default, headline latency, with the cfg4/cfg5 legs); cfg4: 4096 "
                         "instances of M=200 sharded over ranks; cfg5: 400x250 mesh, "
                         "node-partitioned over ranks; cfg2: closed-loop tracking M=100; "
                         "sweep: chain M = 10^3 .. 10^4 device latency")
    ap.add_argument("--batch", type=int, default=4096, help="cfg4 total instances")
    ap.add_argument("--wave", type=int, default=1024, help="cfg4 instances per launch wave")
    ap.add_argument("--cfg5-transport", choices=["torch", "native"], default="torch",
                    help="cfg5 at N > 1: torch.distributed NCCL, or the native NCCL data plane "
                         "(gm_sendrecv / gm_allreduce_sum) with the e2e step captured in one CUDA graph")
    return ap.parse_args()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def problem(M, N):
    from paper_2602_17601_b200 import workloads

    return workloads.scaling_problem(M, N, 0.01, 0)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    return {"hbm_gbs": float(d.get("hbm_gbs") or 6650.0),
            "hbm_note": "of measured" if d.get("hbm_gbs") else "of fallback",
            "sm_mhz": float(d.get("sm_max_mhz") or 1965.0)}


# ---------------------------------------------------------------------------
# the reference's CPU path (baseline/_ref), the oracle port as a fallback
# ---------------------------------------------------------------------------

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


def cpu_oracle_steps(M, N, steps, warmup, threads):
    from threadpoolctl import threadpool_limits

    from oracle import ref_port as O

    topo, model, states, inputs, spec = problem(M, N)
    x0 = states[0]
    times = []
    with threadpool_limits(limits=threads):
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            O.mpc_step(model, topo, spec, x0, np.tile(x0, (N + 1, 1, 1)), np.zeros((N, 6)), N,
                       threads=threads)
            if k >= warmup:
                times.append(time.perf_counter() - t0)
    return float(np.mean(times)) * 1e3


def cpu_step_ms(M, N, steps, warmup, threads):
    """(ms, kind, description) of the reference's CPU step (oracle fallback)."""
    if import_reference() is not None:
        ms = reference_steps(M, N, steps, warmup, threads)[0]
        return ms, "reference", "unmodified reference gnnmpc.mpc.mpc_step (baseline/_ref)"
    return cpu_oracle_steps(M, N, steps, warmup, threads), "port", "oracle mpc_step (baseline/_ref missing)"


def _ref_instance_worker(b):
    """One cfg4 instance through the stock reference mpc_step, 1 BLAS thread
    (multiprocessing worker; the SURVEY 8d cfg4 CPU protocol)."""
    from threadpoolctl import threadpool_limits

    rex, rgr, rm = import_reference()
    from paper_2602_17601_b200 import workloads

    M, N = 200, 20
    topo, model, _, _, spec0 = rex._scaling_problem(M, N, 0.01, 0)
    states, inputs = workloads.batch_instance(b, M, N)
    from gnnmpc.condensing import OcpSpec  # noqa: E402 (reference package on sys.path)

    spec = OcpSpec(topo, N, spec0.q, states[0][:, None, :].repeat(N + 1, axis=1), spec0.r,
                   spec0.u_ref, spec0.input_constraints, spec0.state_constraints)
    cfg = rm.MpcConfig(horizon=N, dt=0.01)
    st = rm.mpc_init(rgr.SystemState(states[0]), cfg, 6)
    st.lin_states = np.concatenate([states, states[-1:]], 0)
    st.lin_inputs = inputs
    with threadpool_limits(limits=1):
        rm.mpc_step(model, topo, spec, rgr.SystemState(states[0]), st, cfg)
    return b


def reference_cfg4(n_inst, procs):
    """solves/s of the stock reference on n_inst cfg4 instances, procs worker
    processes (1 BLAS thread each)."""
    import multiprocessing as mp

    ref = str(ROOT / "baseline" / "_ref")
    sys.path.insert(0, ref)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_ref_instance_worker, range(procs))  # warm-up (imports, first call)
        t0 = time.perf_counter()
        pool.map(_ref_instance_worker, range(n_inst))
        dt = time.perf_counter() - t0
    return n_inst / dt


def reference_arm(args, world, rank):
    """The reference's own CPU implementation of the path, timed on the host
    cores: the unmodified package from baseline/_ref through its public
    mpc_step (BLAS threads = condense threads = all cores); the oracle port
    only if the install is missing.  Rank 0 alone runs at N>1."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    M, N = args.nodes, args.horizon
    status = iters = None
    if args.workload == "cfg4" and import_reference() is not None:
        n_inst = max(cores, 2 * cores)
        v = reference_cfg4(n_inst, cores)
        ms = 1000.0 / v
        kind = "reference"
        what = (f"{n_inst} cfg4 instances (M=200, N=20) through the unmodified reference mpc_step, "
                f"{cores} worker processes x 1 BLAS thread (SURVEY 8d cfg4 protocol)")
        workload = "cfg4: independent chain M=200, N=20 instances"
    elif import_reference() is not None:
        ms, status, iters = reference_steps(M, N, args.steps, args.warmup, cores)
        v = 1000.0 / ms
        kind = "reference"
        what = (f"{args.steps} calls of the unmodified reference gnnmpc.mpc.mpc_step "
                f"(baseline/_ref) after {args.warmup} warm-up, M={M}, N={N}, "
                f"_scaling_problem seed 0, BLAS threads = condense threads = {cores}")
        workload = WORKLOAD
    else:
        ms = cpu_oracle_steps(M, N, args.steps, args.warmup, cores)
        v = 1000.0 / ms
        kind = "port"
        what = (f"{args.steps} oracle mpc_step calls (after {args.warmup} warm-up) at M={M}, "
                f"N={N}, BLAS threads = condense threads = {cores} (baseline/_ref missing)")
        workload = WORKLOAD
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload, "nodes": M, "horizon": N,
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
        """Start sampling every 50 ms; returns once the first sample arrived."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
            return self
        t0 = time.time()
        while not self.lines and time.time() - t0 < wait_s:
            time.sleep(0.02)
        return self

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


def max_over_ranks(values, world, dev):
    if world == 1:
        return [float(v) for v in values]
    import torch

    t = torch.tensor([float(v) for v in values], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def barrier(world):
    if world > 1:
        import torch

        torch.distributed.barrier()


# ---------------------------------------------------------------------------
# algorithmic counts
# ---------------------------------------------------------------------------

def qp_flops(n, m, ng, iters):
    """Algorithmic fp64 flops of the reference's IPM (qpsolver.py:170-229) on
    the expanded QP, per iteration: Schur rank-ng update ng n^2, Cholesky
    n^3/3, two K^{-1} solves 2 x 2n^2, H u 2n^2, the general-row products
    4 ng n (single-nonzero rows are O(m) and left out).  ng = rows with more
    than one nonzero (the soft state rows; the box and slack-sign rows are
    single-nonzero)."""
    per = ng * n * n + n ** 3 / 3.0 + 4.0 * n * n + 2.0 * n * n + 4.0 * ng * n
    return per * max(iters, 1)


def cond_bytes(M, E, N, nx=6, nu=6, B=1):
    """Compulsory fp32 bytes of the Gamma recursion (read stage n once, write
    stage n+1 once, causal columns + Gamma_x) plus its A/B/c blocks."""
    gam = 4.0 * M * nx * sum((1 + k * nu) + (1 + (k + 1) * nu) for k in range(N))
    blocks = N * (M * nx * nx * 4 + E * nx * nx * 4 + M * nx * nu * 4 + M * nx * 8)
    return B * (gam + blocks)


def hg_flops(M, N, nx=6, nu=6, B=1):
    return B * M * sum(2 * nx * nx * k * nu + 2 * nx * (k * nu) ** 2 for k in range(1, N + 1))


FP32_FMA_PER_SM_CLK = 128  # SIMT fp32 FMA lanes per SM per clock (4 SMSPs x 32)


def cond_flops(M, E, N, nx=6, nu=6, B=1):
    """Algorithmic fp32 flops of K-COND: the recursion over the live columns
    (A blocks of node + in-edges times stage-n Gamma: 6n causal + the Gamma_x
    column), Qs Gamma on the causal columns, and H's lower block triangle
    (k(k+1)/2 6x6 pairs over the 6 rows of every node-stage)."""
    rec = sum(2 * nx * nx * (M + E) * (n * nu + 1) for n in range(N))
    qg = M * sum(2 * nx * nx * k * nu for k in range(1, N + 1))
    h = M * sum(2 * nx * nu * nu * k * (k + 1) // 2 for k in range(1, N + 1))
    return B * (rec + qg + h)


def simt_roof(flops, ms, sm_mhz):
    """K-COND against the SIMT fp32 FMA rate (its arithmetic runs on the FMA
    pipe, not the tensor cores: see DESIGN 2 on TMEM accumulation)."""
    peak = 148 * FP32_FMA_PER_SM_CLK * 2 * sm_mhz * 1e6 / 1e12
    ach = flops / (ms * 1e-3) / 1e12
    return {"bound": "fp32 FMA (SIMT)", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": ach / peak, "algorithmic_flops": flops}


def events(n):
    import torch

    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


# ---------------------------------------------------------------------------
# cfg3 (default): latency of one instance per GPU
# ---------------------------------------------------------------------------

def cfg3_leg(args, world, rank, local, dev):
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime
    from paper_2602_17601_b200.mpc import get_plan

    M, N = args.nodes, args.horizon
    topo, model, states, inputs, spec = problem(M, N)
    spec.freeze()
    model.freeze()  # a deployed controller's fixed weights: checked by identity, not re-hashed per step
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    x0 = states[0]
    xs = pkg.SystemState(x0)
    st0 = pkg.MpcState(lin_states=torch.from_numpy(np.tile(x0, (N + 1, 1, 1))).to(dev),
                       lin_inputs=torch.zeros((N, 6), dtype=torch.float64, device=dev))
    for _ in range(3):  # upload, eager run, CUDA-graph capture
        u, st1 = pkg.mpc_step(model, topo, spec, xs, st0, cfg)
    eng = pkg.device.engine(topo, model)
    plan = get_plan(eng, spec, N, 6, 6, cfg, True)
    assert plan.graphs is not None, "plan was not captured as CUDA graphs"
    status, iters = st1.last_status.value, st1.last_iterations
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    L = _runtime.lib()

    for _ in range(args.warmup):
        plan.enqueue(timed=True)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    step_ms, lin_ms, cond_ms, solve_ms = [], [], [], []
    barrier(world)
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
    # end to end through the public API
    for _ in range(args.warmup):
        pkg.mpc_step(model, topo, spec, xs, st0, cfg)
    e2e = []
    for _ in range(args.steps):
        if not args.no_l2_flush:
            flush.fill_(1.0)
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        pkg.mpc_step(model, topo, spec, xs, st0, cfg)
        e2e.append(time.perf_counter() - t0)
    clk = clocks.stop()
    ms, e2e_ms = max_over_ranks([np.mean(step_ms), np.mean(e2e) * 1e3], world, dev)
    # kernels launched per step: one eager (uncaptured) enqueue
    l1 = L.gm_launch_count()
    saved = plan.graphs
    plan.graphs = None
    plan.enqueue(timed=False)
    plan.graphs = saved
    torch.cuda.synchronize()
    kernels_per_step = int(L.gm_launch_count() - l1)
    del flush
    if rank != 0:
        return None
    pk = peaks()
    smax = pk["sm_mhz"] * 1e6
    solve = float(np.mean(solve_ms))
    n, m = plan.n, plan.m
    ng = int(plan.ds.rows.n_st)
    fl = qp_flops(n, m, ng, iters)
    achieved = fl / (solve * 1e-3) / 1e12
    sm_peak = FP64_DFMA_PER_SM_CLK * 2 * smax / 1e12
    dev_peak = 148 * sm_peak
    roof = {"kernel": "k_solve_qp (+k_finish)", "bound": "tensor", "achieved": achieved,
            "peak": sm_peak, "unit": "TFLOP/s", "frac": achieved / sm_peak,
            "frac_device": achieved / dev_peak, "peak_device": dev_peak,
            "traffic": NCU_TRAFFIC["cfg3"]["k_solve_qp"],
            "algorithmic_flops": fl, "qp": {"n": n, "m": m, "general_rows": ng, "iterations": iters},
            "note": "one fp64 CTA per QP on one SM: peak = that SM's fp64 rate (64 DFMA/clk at max "
                    "clock, nominal; no measured fp64 peak), frac_device against all 148 SMs; "
                    "latency-bound (pivot chain of the Cholesky + barrier-separated phases)"}
    cond = float(np.mean(cond_ms))
    cb = cond_bytes(M, int(topo.edge_count), N)
    hfl = hg_flops(M, N)
    lin = float(np.mean(lin_ms))
    stages = {
        "k_condense_tmap": {
            "bound": "hbm", "achieved": cb / (cond * 1e-3) / 1e9, "peak": pk["hbm_gbs"],
            "unit": "GB/s", "frac": cb / (cond * 1e-3) / 1e9 / pk["hbm_gbs"],
            "algorithmic_bytes": cb, "traffic": NCU_TRAFFIC["cfg3"]["k_condense"],
            "h_flops": hfl, "h_tflops": hfl / (cond * 1e-3) / 1e12,
            "compute": simt_roof(cond_flops(M, int(topo.edge_count), N), cond, pk["sm_mhz"]),
            "note": "stage time incl. constraint rows / soft expansion; Gamma is L2-resident at cfg3; "
                    "H and g accumulate in fp32 FMA inside the recursion kernel (round-to-nearest; "
                    "the tcgen05 variant is opt-in, its accumulator truncates)"},
        "linearize": {"ms": lin, "traffic": NCU_TRAFFIC["cfg3"]["linearize"],
                      "kernels": "k_fwd_chain_mma (psi, phi; fp64 DMMA), k_jac_phi_tc, k_jac_psi_tc "
                                 "(tcgen05 3xTF32), k_lin_self, k_lin_c"},
    }
    cpu = None
    if not args.no_cpu_baseline:
        cms, kind, who = cpu_step_ms(M, N, args.cpu_steps, 1, 1)
        cpu = {"value": 1000.0 / cms, "unit": "solves/s", "cores": 1, "kind": kind,
               "sample": f"{args.cpu_steps} calls of the {who} at M={M}, N={N} (1 warm-up), "
                         "BLAS pinned to 1 thread (reference protocol experiments.py:492-528)",
               "ms_per_step": cms}
    return {
        "metric": METRIC, "value": world * 1000.0 / ms, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "hz": 1000.0 / ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (linearize Jacobians, Gamma, H) / f64 (MLP forward, offsets, QP)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": M, "horizon": N, "instances_per_gpu": 1,
                   "parallelism": f"independent instance per GPU x{world}",
                   "model": "random-init weights, frozen (GnnModel.freeze); spec frozen (OcpSpec.freeze)",
                   "l2": "flushed (256 MiB write) between timed steps" if not args.no_l2_flush
                   else "not flushed", "qp": {"n": n, "m": m, "status": status, "iterations": iters}},
        "stage_ms": {"linearize": lin, "condense": cond, "solve_and_epilogue": solve},
        "e2e": {"value": world * 1000.0 / e2e_ms, "unit": "solves/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": M * 6 * 8, "d2h_bytes_per_step": (6 + 2) * 8,
                "path": "paper_2602_17601_b200.mpc_step (public API), host numpy measurement"},
        "gpu_launches": kernels_per_step,
        "gpu_launch_mode": "one CUDA graph per step (e2e); per-stage graph replays (value)",
        "clocks": clk, "roofline": roof, "roofline_stages": stages, "cpu_baseline": cpu,
    }


# ---------------------------------------------------------------------------
# cfg4: 4096 independent instances, sharded over ranks (no collective)
# ---------------------------------------------------------------------------

def cfg4_leg(args, world, rank, local, dev, steps=None, warmup=None):
    """value: device time of all waves with every input resident in HBM (one
    device-to-device load per wave + the kernel chain); e2e: WavePipeline
    from pinned host arrays (H2D of each wave's inputs on a side stream
    under the previous wave's kernels, D2H of u/status)."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime, workloads
    from paper_2602_17601_b200.batch import BatchedMpc, WavePipeline, shard_range

    steps = steps or args.steps
    warmup = warmup or args.warmup
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

    evs = [events(5) for _ in waves]

    def device_step(timed=False):
        for w, ((a, b), d) in enumerate(zip(waves, resident)):
            bm = bm_for(b - a)
            bm.load(*d)
            bm.enqueue(evs[w] if timed else None)

    pipe = WavePipeline(model, topo, spec, cfg, [b - a for a, b in waves])
    for _ in range(warmup):
        device_step()
        pipe.step(host)
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    e0, e1 = events(2)
    ms, stage = [], np.zeros(4)
    for _ in range(steps):
        e0.record()
        device_step(timed=True)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        for ev in evs:
            stage += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    stage /= steps * len(waves)
    t0 = time.perf_counter()
    for _ in range(steps):
        res = pipe.step(host)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) / steps * 1e3
    clk = clocks.stop()
    L = _runtime.lib()
    l1 = L.gm_launch_count()
    device_step()
    torch.cuda.synchronize()
    launches = int(L.gm_launch_count() - l1)
    dev_ms, e2e_ms = max_over_ranks([np.mean(ms), e2e_ms], world, dev)
    if rank != 0:
        return None
    pk = peaks()
    per = hi - lo
    iters = [int(i) for r in res for i in r.iterations]
    wave = waves[0][1] - waves[0][0]
    cb = cond_bytes(M, int(topo.edge_count), N, B=wave)
    cond = float(stage[1])
    cpu = None
    if not args.no_cpu_baseline and import_reference() is not None:
        n_inst = 16
        v = reference_cfg4(n_inst, 1)
        cpu = {"value": v, "unit": "solves/s", "cores": 1, "kind": "reference",
               "sample": f"{n_inst} cfg4 instances through the unmodified reference mpc_step, "
                         "1 process x 1 BLAS thread"}
    return {
        "metric": METRIC, "value": args.batch / (dev_ms * 1e-3), "unit": "solves/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": dev_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": f"cfg4: {args.batch} independent chain M=200, N=20 instances",
                   "instances_per_gpu": per, "wave": args.wave,
                   "parallelism": f"instance shards x{world}, no collective",
                   "l2": "inputs (~1.3 GB per wave set) larger than L2",
                   "qp_iterations_mean_rank0": float(np.mean(iters))},
        "stage_ms_per_wave": {"linearize": float(stage[0]), "condense": cond, "qp": float(stage[2]),
                              "epilogue": float(stage[3])},
        "e2e": {"value": args.batch / (e2e_ms * 1e-3), "unit": "solves/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": per * (M * 6 + (N + 1) * M * 6 + N * 6 + M * (N + 1) * 6) * 8,
                "d2h_bytes_per_step": per * 8 * 8,
                "path": "batch.WavePipeline.step from pinned host arrays (H2D overlapped with the "
                        "previous wave's kernels; wall clock)"},
        "gpu_launches": launches,
        "roofline": {"kernel": "k_condense_tmap (K-COND) + rows/soft", "bound": "hbm",
                     "achieved": cb / (cond * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": cb / (cond * 1e-3) / 1e9 / pk["hbm_gbs"], "algorithmic_bytes": cb,
                     "traffic": NCU_TRAFFIC["cfg4"]["k_condense"],
                     "compute": simt_roof(cond_flops(M, int(topo.edge_count), N, B=wave), cond,
                                          pk["sm_mhz"]),
                     "note": f"per wave of {wave} instances; peak {pk['hbm_note']}"},
        "clocks": clk, "cpu_baseline": cpu,
    }


# ---------------------------------------------------------------------------
# cfg5: 10^5-node mesh, node-partitioned over ranks
# ---------------------------------------------------------------------------

def cfg5_leg(args, world, rank, local, dev, steps=None, warmup=None):
    """400x250 mesh (1e5 nodes), N=20.  world 1: fused persistent
    condensing; world > 1: each rank owns a row slab and keeps owned + halo
    rows only, per-stage NCCL halo exchange of Gamma rows, one all-reduce of
    [H | g | C | d], the QP replicated.  value: device time of the step with
    the trajectory resident; e2e: the measurement (owned + halo rows) from
    pinned host memory each step, D2H of [u, status, iterations]."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime, workloads
    from paper_2602_17601_b200.partition import PartitionedMpc, partition_nodes

    steps = steps or args.steps
    warmup = warmup or args.warmup
    N = 20
    topo, model, states, inputs, spec = workloads.mesh_problem(400, 250, N, 0.01, 0)
    spec.freeze()
    cfg = pkg.MpcConfig(horizon=N, dt=0.01)
    part = partition_nodes(topo, world, rank)
    native = args.cfg5_transport == "native" and world > 1
    transport = None
    if native:
        from paper_2602_17601_b200.partition import NcclTransport

        transport = NcclTransport(rank, world, dev)
    pm = PartitionedMpc(model, topo, spec, cfg, part, transport=transport)
    step_fn = pm.step_graph if native else pm.step
    loc = part.local_nodes if world > 1 else np.arange(topo.node_count)
    ls = torch.from_numpy(np.ascontiguousarray(np.concatenate([states, states[-1:]], 0)[:, loc])).to(dev)
    li = torch.from_numpy(inputs).to(dev)
    x0 = torch.from_numpy(np.ascontiguousarray(states[0][loc])).to(dev)
    xh = torch.from_numpy(np.ascontiguousarray(states[0][loc])).pin_memory()
    for _ in range(warmup):
        pm.step(x0, ls, li)
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    ev = events(5)
    ms, stage = [], np.zeros(4)
    for _ in range(steps):
        pm.load(x0, ls, li)
        pm.enqueue(ev)
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[4]))
        stage += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    stage /= steps
    step_fn(xh, ls, li)  # (captures the step graph on the native path)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        u, st, it = step_fn(xh, ls, li)
    e2e_ms = (time.perf_counter() - t0) / steps * 1e3
    clk = clocks.stop()
    L = _runtime.lib()
    l1 = L.gm_launch_count()
    pm.step(x0, ls, li)
    launches = int(L.gm_launch_count() - l1)
    m, e2e_ms = max_over_ranks([np.mean(ms), e2e_ms], world, dev)
    if rank != 0:
        return None
    pk = peaks()
    M, E = topo.node_count, int(topo.edge_count)
    cb = cond_bytes(M, E, N) / world  # per rank share of the compulsory bytes
    cond = float(stage[1])
    cpu = None
    if not args.no_cpu_baseline and import_reference() is not None:
        # bounded sample: the reference on a 50x40 mesh (2,000 nodes) with
        # the same recipe, scaled linearly to 10^5 nodes (the reference's own
        # measured node-count slope is ~1)
        from threadpoolctl import threadpool_limits

        from paper_2602_17601_b200.graph import mesh_topology  # noqa: F401

        rex, rgr, rm = import_reference()
        t_s, m_s = _reference_mesh_step(50, 40, N)
        scale = M / m_s
        cpu = {"value": 1.0 / (t_s * scale), "unit": "solves/s", "cores": 1, "kind": "reference",
               "sample": f"one unmodified reference mpc_step on a 50x40 mesh ({m_s} nodes, cfg5 "
                         f"recipe) = {t_s * 1e3:.0f} ms, scaled linearly x{scale:.0f} to 10^5 nodes, "
                         "1 BLAS thread", "measured_s": t_s}
    return {
        "metric": METRIC, "value": 1000.0 / m, "unit": "solves/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": m, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": "cfg5: 2D mesh 400x250 = 100000 nodes, horizon 20",
                   "parallelism": (f"node partition x{world} (row slabs, owned + halo rows per rank), "
                                   "NCCL halo per stage + one all-reduce" if world > 1
                                   else "single GPU, fused persistent recursion + cost"),
                   "l2": "working set (Gamma 1.07 GB) larger than L2",
                   "transport": (("native NCCL (gm_sendrecv / gm_allreduce_sum), e2e step as one CUDA "
                                  "graph" if native else "torch.distributed NCCL") if world > 1 else None),
                   "qp": {"status": st, "iterations": it}},
        "stage_ms": {"linearize": float(stage[0]), "condense_incl_exchange": cond,
                     "qp": float(stage[2]), "epilogue": float(stage[3])},
        "e2e": {"value": 1000.0 / e2e_ms, "unit": "solves/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(len(loc)) * 6 * 8, "d2h_bytes_per_step": 64,
                "path": "PartitionedMpc.step: measurement H2D from pinned host memory, trajectory "
                        "device-resident between steps (like MpcState), D2H of u/status"},
        "gpu_launches": launches,
        "roofline": {"kernel": "condensing (K-COND k_condense_tmap at 1 GPU; K-REC stages + K-HG when "
                               "partitioned)", "bound": "hbm",
                     "achieved": cb / (cond * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": cb / (cond * 1e-3) / 1e9 / pk["hbm_gbs"], "algorithmic_bytes": cb,
                     "traffic": NCU_TRAFFIC["cfg5"]["k_condense"],
                     "compute": simt_roof(cond_flops(M, E, N) / world, cond, pk["sm_mhz"]),
                     "note": f"rank 0's share of the compulsory Gamma + block bytes; peak {pk['hbm_note']}"},
        "clocks": clk, "cpu_baseline": cpu,
    }


def _reference_mesh_step(rows, cols, N):
    """One stock reference mpc_step on the cfg5 recipe at rows x cols
    (seconds, node count), 1 BLAS thread."""
    from threadpoolctl import threadpool_limits

    rex, rgr, rm = import_reference()
    from paper_2602_17601_b200 import workloads

    topo_o, model_o, states, inputs, spec_o = workloads.mesh_problem(rows, cols, N, 0.01, 0)
    import gnnmpc.condensing as rc  # reference (on sys.path via import_reference's package)
    import gnnmpc.gnn as rg

    topo = rgr.GraphTopology(topo_o.node_count, topo_o.in_neighbors, topo_o.neighbor_bound)

    def mlp(p):
        import gnnmpc.mlp as rmlp
        return rmlp.MlpParams(list(p.layer_dims), [w.copy() for w in p.weights], [b.copy() for b in p.biases])

    nrm = model_o.normalization
    model = rg.GnnModel(mlp(model_o.psi), mlp(model_o.phi), model_o.dt, model_o.n_p, model_o.n_u,
                        model_o.n_m, rg.Normalization(nrm.state_mean, nrm.state_scale, nrm.input_mean,
                                                      nrm.input_scale))
    spec = rc.OcpSpec(topo, N, spec_o.q, spec_o.x_ref, spec_o.r, spec_o.u_ref,
                      list(spec_o.input_constraints),
                      [rc.StateConstraint(s.node, s.stage, s.c, s.d, s.soft, s.rho1, s.rho2)
                       for s in spec_o.state_constraints])
    cfg = rm.MpcConfig(horizon=N, dt=0.01)
    x = rgr.SystemState(states[0])
    st = rm.mpc_init(x, cfg, 6)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        rm.mpc_step(model, topo, spec, x, st, cfg)
        t = time.perf_counter() - t0
    return t, topo.node_count


# ---------------------------------------------------------------------------
# cfg2: closed-loop tracking (replicas)
# ---------------------------------------------------------------------------

def cfg2_leg(args, world, rank, local, dev):
    """Closed-loop tracking, chain M=100 (BASELINE cfg2): ChainConfig(100),
    settled 3 s, end effector on a 0.04 m / 8 s circle around its settled
    position, default TrackingWeights, random-init GNN (no training data),
    horizon 20.  A step = one controller step (mpc_step) + one plant period
    (device kernel); the state stays on the device, per step x_ref (H2D) and
    [u, status, iterations] (D2H) cross."""
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200 import _runtime
    from paper_2602_17601_b200.graph import chain_topology
    from paper_2602_17601_b200.tracking import (TrackingWeights, circle_reference,
                                                 run_closed_loop_device, tracking_spec_provider)
    from paper_2602_17601_b200.trunk import ChainConfig, DevicePlant

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
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    L = _runtime.lib()
    l1 = L.gm_launch_count()
    t0 = time.perf_counter()
    log = run_closed_loop_device(plant, model, topo, prov, x0, args.steps, cfg)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / args.steps * 1e3
    launches = int((L.gm_launch_count() - l1) / args.steps)
    clk = clocks.stop()
    ms, = max_over_ranks([ms], world, dev)
    if rank != 0:
        return None
    tm = log.timings.mean(axis=0)
    cpu = None
    if not args.no_cpu_baseline:
        cms, kind, what = _cpu_closed_loop(M, N, x0.cpu().numpy(), center, max(2, min(args.cpu_steps, 6)))
        cpu = {"value": 1000.0 / cms, "unit": "steps/s", "cores": 1, "kind": kind, "sample": what,
               "ms_per_step": cms}
    return {
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
        "gpu_launches": launches,
        "roofline": {"kernel": "k_solve_qp", "bound": "tensor", "achieved": None,
                     "peak": FP64_DFMA_PER_SM_CLK * 2 * peaks()["sm_mhz"] * 1e6 / 1e12, "unit": "TFLOP/s",
                     "frac": None, "traffic": None,
                     "note": "wall-clock closed loop; the QP (one fp64 CTA) dominates the device time "
                             "(stage_ms); see the cfg3 line for its roofline"},
        "clocks": clk, "cpu_baseline": cpu,
    }


def _cpu_closed_loop(M, N, x0, center, n_steps):
    """The reference's own closed loop (run_closed_loop with its plant and
    tracking provider) when installed, else the oracle's; ms per step."""
    from threadpoolctl import threadpool_limits

    ref = import_reference()
    if ref is not None:
        rex, rgr, rm = ref
        import gnnmpc.gnn as rg
        import gnnmpc.references as rr
        import gnnmpc.trunk as rt

        pc = rt.ChainConfig(node_count=M)
        topo = rgr.chain_topology(M)
        model = rg.init_model(3, 6, 0.01, np.random.default_rng(0), out_scale=0.05)
        cfg = rm.MpcConfig(horizon=N, dt=0.01)
        xs = rgr.SystemState(x0)
        prov = rex.tracking_spec_provider(topo, cfg, xs, rr.circle_reference(0.04, 8.0, center),
                                          rex.TrackingWeights(), pc.n_u, pc.u_max)
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            rm.run_closed_loop(rex.make_plant_step(pc), model, topo, prov, xs, n_steps, cfg)
            ms = (time.perf_counter() - t0) / n_steps * 1e3
        return ms, "reference", (f"{n_steps} closed-loop steps of the unmodified reference "
                                 f"run_closed_loop (its trunk plant and tracking provider) at M={M}, "
                                 f"N={N}, 1 BLAS thread")
    from oracle import ref_port as O
    import paper_2602_17601_b200 as pkg

    model = pkg.init_model(3, 6, 0.01, np.random.default_rng(0), out_scale=0.05)
    from paper_2602_17601_b200.graph import chain_topology

    topo = chain_topology(M)
    P = O.trunk_params(M)
    specs = O.tracking_specs(topo, N, 0.01, x0, O.circle_ref(0.04, 8.0, center), 6, 8.0)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        O.closed_loop(model, topo, P, specs, x0, n_steps, N)
        ms = (time.perf_counter() - t0) / n_steps * 1e3
    return ms, "port", f"{n_steps} oracle closed-loop steps at M={M}, N={N}, 1 BLAS thread"


# ---------------------------------------------------------------------------
# sweep: near-constant latency up to 10^4 nodes (north_star)
# ---------------------------------------------------------------------------

def sweep_leg(args, world, rank, local, dev):
    import torch

    import paper_2602_17601_b200 as pkg
    from paper_2602_17601_b200.mpc import get_plan

    out = []
    clocks = ClockSampler(local).start()
    N = args.horizon
    for M in (1000, 2000, 5000, 10000):
        topo, model, states, inputs, spec = problem(M, N)
        spec.freeze()
        cfg = pkg.MpcConfig(horizon=N, dt=0.01)
        xs = pkg.SystemState(states[0])
        st0 = pkg.mpc_init(xs, cfg, 6)
        for _ in range(3):
            u, st1 = pkg.mpc_step(model, topo, spec, xs, st0, cfg)
        plan = get_plan(pkg.device.engine(topo, model), spec, N, 6, 6, cfg, True)
        for _ in range(args.warmup):
            plan.enqueue(timed=True)
        torch.cuda.synchronize()
        ms, st = [], np.zeros(3)
        for _ in range(args.steps):
            plan.enqueue(timed=True)
            torch.cuda.synchronize()
            st += plan.stage_ms()
            ms.append(plan.events[0].elapsed_time(plan.events[3]))
        st /= args.steps
        out.append({"nodes": M, "ms_per_step": float(np.mean(ms)), "linearize": float(st[0]),
                    "condense": float(st[1]), "qp_and_epilogue": float(st[2]),
                    "qp_status": st1.last_status.value, "qp_iterations": st1.last_iterations})
    clk = clocks.stop()
    if rank != 0:
        return None
    m0, m1 = out[0]["ms_per_step"], out[-1]["ms_per_step"]
    return {"metric": METRIC, "value": 1000.0 / m1, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m1, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": "sweep: chain M = 1e3 .. 1e4, N = 20 (value at M = 1e4)"},
            "sweep": out, "latency_ratio_1e4_vs_1e3": m1 / m0, "clocks": clk}


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    try:
        if args.workload == "cfg2":
            out = cfg2_leg(args, world, rank, local, dev)
        elif args.workload == "cfg4":
            out = cfg4_leg(args, world, rank, local, dev)
        elif args.workload == "cfg5":
            out = cfg5_leg(args, world, rank, local, dev)
        elif args.workload == "sweep":
            out = sweep_leg(args, world, rank, local, dev)
        else:
            out = cfg3_leg(args, world, rank, local, dev)
            if not args.no_legs:
                legs = {}
                ls, lw = min(args.steps, 5), max(3, min(args.warmup, 3))
                for name, fn in (("cfg4", cfg4_leg), ("cfg5", cfg5_leg)):
                    try:
                        legs[name] = fn(args, world, rank, local, dev, steps=ls, warmup=lw)
                    except Exception as e:  # a leg must never hide the headline line
                        legs[name] = {"error": f"{type(e).__name__}: {e}"}
                if out is not None:
                    out["legs"] = legs
        if out is not None:
            print(json.dumps(out), flush=True)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
