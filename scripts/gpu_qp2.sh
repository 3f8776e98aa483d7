timeout 300 python scripts/qp_phases.py cfg3 2>&1 | tail -17
