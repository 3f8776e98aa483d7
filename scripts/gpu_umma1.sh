timeout 300 python -m pytest tests/test_gpu_umma.py -x -q -p no:cacheprovider > gpurun_out/umma.log 2>&1; echo "umma rc=$?"; tail -15 gpurun_out/umma.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_cfg5.csv | head -14
