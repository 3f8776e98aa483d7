timeout 200 python -m pytest tests/test_gpu_stages.py -m gpu -q -p no:cacheprovider -k "cholesky or random_qps" 2>&1 | tail -25
timeout 100 python scripts/qp_phases.py cfg3 2>&1 | tail -14
