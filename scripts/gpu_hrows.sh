# K-QP h_apply row-per-thread on on-chip H, u gathered once: GPU tests, QP phases at cfg3, default bench, cfg4 bench
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; head -16 gpurun_out/qp_phases.txt
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-steps 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['stage_ms'], d['e2e']['ms_per_step'], d['config']['qp'])"
timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_cfg4.json; echo "bench cfg4: $(python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print(d['ms_per_step'], d['value'], d['e2e']['value'])")"
