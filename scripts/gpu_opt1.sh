set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 5 2>&1 | tail -6
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_opt1.json 2> gpurun_out/bench_opt1.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_opt1.json
