timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_stages.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/pytest_gh.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_gh.log | head -10
for gh in 256 128; do for q in 0 4 6; do for w in cfg4; do GM_TMA_GH=$gh GM_TMA_QGR=$q timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_${w}.json 2> gpurun_out/b.err; python -c "
import json;d=json.loads(open('gpurun_out/b_${w}.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave'));print('gh $gh qgr $q $w', round(d['ms_per_step'],3), s.get('condense', s.get('condense_incl_exchange')))"; done; done; done
for gh in 256 128; do GM_TMA_GH=$gh timeout 300 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b5.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b5.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave'));print('gh $gh cfg5', round(d['ms_per_step'],3), s)"
GM_TMA_GH=$gh timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('gh $gh cfg3', round(d['ms_per_step'],3), d['stage_ms']['condense'])"; done
