timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
python scripts/profile_stages.py --M 1000 --N 20 --reps 5 2>&1 | tail -3
python scripts/profile_stages.py --M 10 --N 10 --reps 3 2>&1 | tail -2
