timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print("cfg3", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3), {k: round(v,3) for k,v in d["stage_ms"].items()}, "launches", d["gpu_launches"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k, v in d.get("legs", {}).items():
    if "error" in v: print(k, v); continue
    s = v.get("stage_ms", v.get("stage_ms_per_wave"))
    print(k, round(v["ms_per_step"],3), round(v["value"],1), v["unit"], "e2e", round(v["e2e"]["ms_per_step"],3), {a: round(b,3) for a,b in s.items()}, "roof", round(v["roofline"]["frac"],4), v["clocks"]["reasons"])
PY
