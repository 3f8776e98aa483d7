timeout 100 python scripts/qp_phases.py cfg1_chain10 cfg3 2>&1 | tail -30
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 120 python scripts/profile_stages.py --M 1000 --N 20 --reps 4 2>&1 | tail -2
