timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b5.json; python -c "import json;d=json.load(open('gpurun_out/b5.json'));print('cfg5', d['ms_per_step'])"
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b4.json; python -c "import json;d=json.load(open('gpurun_out/b4.json'));print('cfg4', d['ms_per_step'], d['value'])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b3.json; python -c "import json;d=json.load(open('gpurun_out/b3.json'));print('cfg3', d['ms_per_step'], d['stage_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_condense_tc -c 2 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E 'duration' | head -3
