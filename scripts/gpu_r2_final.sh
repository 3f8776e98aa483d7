# round-2 final evidence: GPU suite, smoke, benches, launch lists, ncu --set full of the dominant kernels
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --workload sweep --steps 10 --warmup 3 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo "sweep rc=$?"
timeout 900 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print("cfg3", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3), {k: round(v,3) for k,v in d["stage_ms"].items()}, "launches", d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k, v in d.get("legs", {}).items():
    if "error" in v: print(k, v); continue
    s = v.get("stage_ms", v.get("stage_ms_per_wave"))
    print(k, round(v["ms_per_step"],3), round(v["value"],1), v["unit"], "e2e", round(v["e2e"]["ms_per_step"],3), {a: round(b,3) for a,b in s.items()}, "roof", round(v["roofline"]["frac"],4), v["clocks"]["reasons"])
PY
# launch lists (cold, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-legs > /dev/null 2>&1; echo "ncu launches cfg3 rc=$?"
for w in cfg4 cfg5; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches $w rc=$?"; done
# full captures: cfg3 kernels; K-COND at cfg4 / cfg5
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_solve_qp|k_condense_tmap|k_fwd_chain_mma|k_jac_phi_tc|k_jac_psi_tc|k_lin_self|k_lin_c" -c 8 -o gpurun_out/full_cfg3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-legs > /dev/null 2>&1; echo "ncu full cfg3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_condense_tmap|k_rollout" -c 2 -o gpurun_out/full_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full cfg4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_condense_tmap|k_rollout" -c 2 -o gpurun_out/full_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full cfg5 rc=$?"
ls -la gpurun_out/*.csv gpurun_out/*.ncu-rep
