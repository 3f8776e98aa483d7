timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py tests/test_gpu_local.py -q -p no:cacheprovider -x > gpurun_out/pytest_q5.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_q5.log | head -10
for w in cfg4 cfg5; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_${w}.json 2> gpurun_out/b.err; python -c "
import json;d=json.loads(open('gpurun_out/b_${w}.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave'));print('$w', round(d['ms_per_step'],3), s)"; done
timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('cfg3', round(d['ms_per_step'],3), d['stage_ms']['condense'])"
