timeout 300 python -m pytest tests/test_gpu_fused.py tests/test_gpu_stages.py -q -p no:cacheprovider -x > gpurun_out/pytest_q4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_q4.log
timeout 300 python scripts/cond_stages.py > gpurun_out/cond_stages.txt 2>&1; cat gpurun_out/cond_stages.txt | cut -c1-130
for w in cfg4; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_${w}.json 2> gpurun_out/b.err; python -c "
import json;d=json.loads(open('gpurun_out/b_${w}.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave'));print('$w', round(d['ms_per_step'],3), s)"; done
