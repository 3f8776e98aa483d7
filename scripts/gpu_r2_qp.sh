# K-QP iteration: QP-related GPU tests, cfg3 bench, phase profile
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/pytest_qp.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E " gpurun_out/pytest_qp.log | head -20
timeout 300 python bench.py --no-legs --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bench_qp.json 2> gpurun_out/bench_qp.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_qp.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['stage_ms'], d['config']['qp'])"
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; cat gpurun_out/qp_phases.txt
timeout 300 python scripts/qp_phases.py cfg3 --chol > gpurun_out/qp_phases_chol.txt 2>&1; tail -4 gpurun_out/qp_phases_chol.txt
