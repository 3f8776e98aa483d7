timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; cat gpurun_out/qp_phases.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b3.json; python -c "import json;d=json.load(open('gpurun_out/b3.json'));print(d['ms_per_step'], d['stage_ms'], d['config']['qp'], d['e2e']['ms_per_step'])"
