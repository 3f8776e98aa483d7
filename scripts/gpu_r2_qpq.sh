timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_reference_dropin.py -q -p no:cacheprovider -x > gpurun_out/pytest_qpq.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_qpq.log | head -10
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; cat gpurun_out/qp_phases.txt
for i in 1 2; do timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('cfg3', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['e2e']['ms_per_step'],3))"; done
