python scripts/qp_one.py cfg1_chain10 2 > gpurun_out/qp_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_solve_qp -c 1 -o gpurun_out/qp_prof python scripts/qp_one.py cfg1_chain10 1 > gpurun_out/qp_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/qp_ncu.log
