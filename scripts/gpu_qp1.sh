timeout 600 python -m pytest tests/test_gpu_stages.py -x -q -k "qp or chol or mpc_step" 2>&1 | tail -3
timeout 300 python scripts/qp_phases.py cfg3 2>&1 | tail -20
timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 4 2>&1 | tail -2
