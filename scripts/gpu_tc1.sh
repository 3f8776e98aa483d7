timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_umma.py -x -q -p no:cacheprovider > gpurun_out/tc.log 2>&1; echo "tc rc=$?"; tail -30 gpurun_out/tc.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"; cat gpurun_out/bench_cfg5.json
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "cfg3 rc=$?"; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.txt; head -8 gpurun_out/launches_cfg5.txt
