timeout 300 python scripts/qp_batch148.py && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_qp -s 1 -c 1 -o gpurun_out/full_qp148 python scripts/qp_batch148.py > gpurun_out/ncuqp148.log 2>&1; echo "ncu rc=$?"
