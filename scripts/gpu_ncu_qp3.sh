timeout 120 python scripts/qp_cfg3.py 1 > gpurun_out/qp3_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_qp -c 1 -o gpurun_out/qp3_prof python scripts/qp_cfg3.py 1 > gpurun_out/qp3_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/qp3_ncu.log
