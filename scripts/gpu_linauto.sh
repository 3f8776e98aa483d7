timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b3.json; python -c "import json;d=json.load(open('gpurun_out/b3.json'));print('cfg3', d['ms_per_step'], d['stage_ms'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b2.json; python -c "import json;d=json.load(open('gpurun_out/b2.json'));print('cfg2', d['ms_per_step'], d['stage_ms'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
