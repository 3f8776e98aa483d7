timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py -q -p no:cacheprovider -x > gpurun_out/pytest_gr.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_gr.log | head -10
for gr in 0 128 256; do for w in cfg4 cfg5; do GM_TMA_GR=$gr timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_${w}.json 2> gpurun_out/b.err; python -c "
import json;d=json.loads(open('gpurun_out/b_${w}.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave'));print('gr $gr $w', round(d['ms_per_step'],3), s.get('condense', s.get('condense_incl_exchange')))"; done; done
GM_TMA_GR=256 timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('gr 256 cfg3', round(d['ms_per_step'],3), d['stage_ms']['condense'])"
timeout 300 python scripts/cond_stages.py mesh > gpurun_out/cond_stages_mesh.txt 2>&1; cat gpurun_out/cond_stages_mesh.txt
