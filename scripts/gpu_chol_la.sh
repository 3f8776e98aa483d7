timeout 300 python -m pytest tests/test_gpu_stages.py -q -p no:cacheprovider -k "cholesky" 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; head -8 gpurun_out/qp_phases.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b3.json; python -c "import json;d=json.load(open('gpurun_out/b3.json'));print('cfg3', d['ms_per_step'], d['stage_ms'], d['config']['qp'], d['e2e']['ms_per_step'])"
