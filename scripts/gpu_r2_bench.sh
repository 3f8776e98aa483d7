# round-2 bench: default line (cfg3 + cfg4/cfg5 legs), cfg2, sweep, reference arm
( time timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2> gpurun_out/bench_default.time; echo "default rc=$?"; cat gpurun_out/bench_default.time | grep real
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print("cfg3", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3), d["stage_ms"], "launches", d["gpu_launches"])
print("roof", {k: d["roofline"][k] for k in ("achieved","peak","frac","frac_device")})
print("cpu", d["cpu_baseline"])
for k, v in d.get("legs", {}).items():
    if "error" in v: print(k, v); continue
    print(k, round(v["ms_per_step"],3), v["value"], v["unit"], "e2e", round(v["e2e"]["ms_per_step"],3), v.get("stage_ms", v.get("stage_ms_per_wave")), "roof", round(v["roofline"]["frac"],4), "cpu", v.get("cpu_baseline"))
PY
timeout 600 python bench.py --workload cfg2 --steps 20 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"; tail -c 400 gpurun_out/bench_cfg2.json
timeout 600 python bench.py --workload sweep --steps 10 --warmup 3 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo "sweep rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_sweep.json').read().strip().splitlines()[-1]);print([(s['nodes'],round(s['ms_per_step'],3),s['qp_iterations']) for s in d['sweep']])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
