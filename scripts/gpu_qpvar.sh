L=paper_2602_17601_b200/lib
cp $L/libgnnmpc_b200.so /tmp/base.so
for v in t128 t512; do
  cp $L/libgnnmpc_b200_$v.so $L/libgnnmpc_b200.so
  echo "== $v"; timeout 300 python scripts/qp_phases.py cfg3 2>&1 | head -1
  timeout 300 python -m pytest tests/test_gpu_stages.py -q -x -k "qp or cholesky" -p no:cacheprovider 2>&1 | tail -1
done
cp /tmp/base.so $L/libgnnmpc_b200.so
