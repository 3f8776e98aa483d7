timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-legs > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_qp -c 1 -o gpurun_out/full_qp_cfg3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-legs > gpurun_out/ncuqp.log 2>&1; echo "ncu rc=$?"
