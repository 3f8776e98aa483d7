timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for m in 0 3; do GM_LINEARIZE_MODE=$m timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b5_$m.json; python -c "import json;d=json.load(open('gpurun_out/b5_$m.json'));print('cfg5 mode $m', d['ms_per_step'], d['config']['qp'])"; done
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b4.json; python -c "import json;d=json.load(open('gpurun_out/b4.json'));print('cfg4', d['ms_per_step'], d['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.txt; head -16 gpurun_out/launches_cfg5.txt
