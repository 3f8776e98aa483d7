"""Node-count scaling sweep and the ``trunkctl scaling`` report, from the B200
path.

Mirrors ``gnnmpc.experiments.run_scaling_sweep`` / ``loglog_slope``
(``experiments.py:505-578``) and ``gnnmpc.cli.cmd_scaling`` /
``_write_summary`` (``cli.py:263-299``, ``:31-46``): same instance recipe
(``workloads.scaling_problem`` = ``_scaling_problem``), same calls in the same
order, same medians, same ``scaling.csv`` columns and ``summary.json`` keys,
so the two harnesses' outputs compare line by line.

Differences, all stated in the report:

* ``run_scaling_sweep`` times the public API exactly like the reference
  (``linearize_trajectory``; ``condense_gammas`` + ``condense_ocp``;
  ``expand_soft_constraints`` + ``solve_qp``), with a device synchronisation
  before each clock read.  Those calls return NumPy arrays, so the numbers
  include the device-to-host copies of Gamma (M x (N+1) x 6 x N*6 doubles).
* ``condense_peak_mb`` is the peak of the torch CUDA allocator during one
  untimed condense pass (the reference samples host ``tracemalloc``).
* ``run_device_sweep`` adds the operational numbers: the per-stage device
  times of ``mpc_step`` (``StepTiming``), inputs resident on the GPU.
* ``threads`` is accepted and ignored (the GPU path has no thread pool); the
  "multi" columns are therefore not produced.
"""

from __future__ import annotations

import hashlib
import json
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import workloads


@dataclass(frozen=True)
class ScalingRow:
    """``experiments.py:457-462``."""

    node_count: int
    linearize_ms: float
    condense_ms: float
    solve_ms: float
    condense_peak_mb: float


def loglog_slope(x, y) -> float:
    """Least-squares slope of log y against log x (``experiments.py:575-578``)."""
    x = np.log(np.asarray(x, dtype=float))
    y = np.log(np.asarray(y, dtype=float))
    return float(np.polyfit(x, y, 1)[0])


def _sync():
    import torch

    torch.cuda.synchronize()


def run_scaling_sweep(m_list, horizon: int = 20, dt: float = 0.01, reps: int = 3, threads: int = 1,
                      seed: int = 0, solve: bool = True) -> list[ScalingRow]:
    """Condensing time and peak memory versus node count through the public
    API (``experiments.py:505-572``); medians of ``reps`` after a warm-up."""
    import torch

    from .condensing import condense_gammas, condense_ocp, expand_soft_constraints
    from .gnn import linearize_trajectory
    from .qpsolver import QpProblem, SolverSettings, solve_qp

    rows = []
    for M in m_list:
        topo, model, states, inputs, spec = workloads.scaling_problem(int(M), horizon, dt, seed)
        x0 = states[0]
        lin = linearize_trajectory(model, topo, states, inputs)  # warm-up
        gammas = condense_gammas(lin, x0, threads=threads)
        condense_ocp(spec, lin, x0, threads=threads, gammas=gammas)
        _sync()

        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        g2 = condense_gammas(lin, x0, threads=threads)
        condense_ocp(spec, lin, x0, threads=threads, gammas=g2)
        _sync()
        peak = torch.cuda.max_memory_allocated() - base
        del g2

        lin_t, cond_t, solve_t = [], [], []
        for _ in range(reps):
            _sync()
            t0 = time.perf_counter()
            lin = linearize_trajectory(model, topo, states, inputs)
            _sync()
            lin_t.append(time.perf_counter() - t0)

            t0 = time.perf_counter()
            gammas = condense_gammas(lin, x0, threads=threads)
            qp = condense_ocp(spec, lin, x0, threads=threads, gammas=gammas)
            _sync()
            cond_t.append(time.perf_counter() - t0)

            if solve:
                h, g, c, d, _ = expand_soft_constraints(qp)
                _sync()
                t0 = time.perf_counter()
                solve_qp(QpProblem(h, g, c, d), SolverSettings(tolerance=1e-8))
                _sync()
                solve_t.append(time.perf_counter() - t0)
        rows.append(ScalingRow(
            node_count=int(M),
            linearize_ms=float(np.median(lin_t) * 1e3),
            condense_ms=float(np.median(cond_t) * 1e3),
            solve_ms=float(np.median(solve_t) * 1e3) if solve_t else 0.0,
            condense_peak_mb=float(max(peak, 0) / 2**20),
        ))
    return rows


def run_device_sweep(m_list, horizon: int = 20, dt: float = 0.01, reps: int = 3, seed: int = 0):
    """Per-stage device times (``StepTiming``, ``mpc.py:51-56``) of one
    ``mpc_step`` per node count, medians of ``reps`` after a warm-up step."""
    from . import mpc as _mpc
    from .graph import SystemState

    out = []
    for M in m_list:
        topo, model, states, inputs, spec = workloads.scaling_problem(int(M), horizon, dt, seed)
        spec.freeze()
        cfg = _mpc.MpcConfig(horizon=horizon, dt=dt)
        x = SystemState(states[0])
        st = _mpc.mpc_init(x, cfg, 6)
        _mpc.mpc_step(model, topo, spec, x, st, cfg)
        lin_t, cond_t, sol_t, tot_t = [], [], [], []
        for _ in range(reps):
            _, st1 = _mpc.mpc_step(model, topo, spec, x, st, cfg)
            tm = st1.last_timing
            lin_t.append(tm.linearize_ms)
            cond_t.append(tm.condense_ms)
            sol_t.append(tm.solve_ms)
            tot_t.append(tm.linearize_ms + tm.condense_ms + tm.solve_ms)
        out.append({"node_count": int(M), "linearize_ms": float(np.median(lin_t)),
                    "condense_ms": float(np.median(cond_t)), "solve_ms": float(np.median(sol_t)),
                    "step_ms": float(np.median(tot_t)), "status": st1.last_status.value,
                    "iterations": int(st1.last_iterations)})
    return out


def config_hash(cfg: dict) -> str:
    """``cli.py:31-33``."""
    canon = json.dumps(cfg, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(canon.encode()).hexdigest()[:16]


def write_summary(out: Path, command: str, cfg: dict, seed: int, metrics: dict, artifacts: list[str]):
    """``cli.py:36-46``: summary.json with the reference's keys."""
    summary = {"command": command, "config_hash": config_hash(cfg), "seed": seed, "metrics": metrics,
               "artifacts": artifacts}
    with open(Path(out) / "summary.json", "w") as f:
        json.dump(summary, f, indent=1)
    return summary


def write_scaling_csv(path: Path, rows_by_threads) -> None:
    """``scaling.csv`` in the reference's column order (``cli.py:275-283``)."""
    with open(path, "w") as f:
        f.write("node_count,threads,linearize_ms,condense_ms,solve_ms,condense_peak_mb\n")
        for rows, th in rows_by_threads:
            if rows is None:
                continue
            for r in rows:
                f.write(f"{r.node_count},{th},{r.linearize_ms:.6g},{r.condense_ms:.6g},"
                        f"{r.solve_ms:.6g},{r.condense_peak_mb:.6g}\n")


def scaling_metrics(rows_single, device_rows=None) -> dict:
    """``cli.py:284-299`` metrics (single-thread keys), plus the device sweep."""
    ms = [r.node_count for r in rows_single]
    metrics = {
        "m_list": list(map(int, ms)),
        "condense_ms_single": [r.condense_ms for r in rows_single],
        "condense_time_slope_single": loglog_slope(ms, [r.condense_ms for r in rows_single]),
        "condense_memory_slope": loglog_slope(ms, [max(r.condense_peak_mb, 1e-9) for r in rows_single]),
        "linearize_ms_single": [r.linearize_ms for r in rows_single],
        "solve_ms_single": [r.solve_ms for r in rows_single],
    }
    if device_rows:
        dm = [d["node_count"] for d in device_rows]
        metrics["device"] = {
            "linearize_ms": [d["linearize_ms"] for d in device_rows],
            "condense_ms": [d["condense_ms"] for d in device_rows],
            "solve_ms": [d["solve_ms"] for d in device_rows],
            "step_ms": [d["step_ms"] for d in device_rows],
            "step_time_slope": loglog_slope(dm, [d["step_ms"] for d in device_rows]),
            "condense_time_slope": loglog_slope(dm, [d["condense_ms"] for d in device_rows]),
        }
    return metrics


def cmd_scaling(cfg: dict, out: Path, seed: int, threads: int = 1) -> dict:
    """``trunkctl scaling`` (``cli.py:263-299``) on the B200 path: writes
    ``scaling.csv`` (public-API protocol), ``scaling_device.csv`` (device stage
    times of ``mpc_step``) and ``summary.json``; returns the metrics."""
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    m_list = cfg.get("m_list", [16, 32, 64, 128, 256, 512, 1024])
    reps = int(cfg.get("reps", 3))
    horizon = int(cfg.get("horizon", 20))
    rows_single = run_scaling_sweep(m_list, horizon=horizon, reps=reps, threads=1, seed=seed)
    dev = run_device_sweep(m_list, horizon=horizon, reps=reps, seed=seed)
    write_scaling_csv(out / "scaling.csv", [(rows_single, 1)])
    with open(out / "scaling_device.csv", "w") as f:
        f.write("node_count,linearize_ms,condense_ms,solve_ms,step_ms,status,iterations\n")
        for d in dev:
            f.write(f"{d['node_count']},{d['linearize_ms']:.6g},{d['condense_ms']:.6g},{d['solve_ms']:.6g},"
                    f"{d['step_ms']:.6g},{d['status']},{d['iterations']}\n")
    metrics = scaling_metrics(rows_single, dev)
    write_summary(out, "scaling", cfg, seed, metrics, ["scaling.csv", "scaling_device.csv"])
    return metrics


def main(argv=None) -> int:
    import argparse

    ap = argparse.ArgumentParser(description="trunkctl-compatible scaling report from the B200 path")
    ap.add_argument("command", choices=["scaling"])
    ap.add_argument("--config", type=Path, default=None, help="JSON config (m_list, reps, horizon)")
    ap.add_argument("--out", type=Path, required=True)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--threads", type=int, default=1)
    a = ap.parse_args(argv)
    cfg = json.loads(a.config.read_text()) if a.config else {}
    metrics = cmd_scaling(cfg, a.out, a.seed, a.threads)
    print(json.dumps(metrics, indent=1))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
