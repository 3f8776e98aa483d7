timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -5
timeout 300 python scripts/qp_phases.py cfg3 2>&1 | tail -17
timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 4 2>&1 | tail -2
