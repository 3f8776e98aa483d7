timeout 200 python -m pytest tests/test_gpu_stages.py -m gpu -x -q -p no:cacheprovider -k "cholesky or qp" 2>&1 | tail -4
timeout 100 python scripts/qp_phases.py cfg3 2>&1 | tail -17
