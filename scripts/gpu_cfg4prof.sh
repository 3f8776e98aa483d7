timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_cfg4.csv > gpurun_out/launches_cfg4.txt; head -24 gpurun_out/launches_cfg4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.txt; head -24 gpurun_out/launches_cfg5.txt
