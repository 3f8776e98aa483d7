timeout 900 python scripts/diag_precision.py 100 100 2>&1 | tail -6
timeout 900 python scripts/diag_precision.py 40 25 2>&1 | tail -6
