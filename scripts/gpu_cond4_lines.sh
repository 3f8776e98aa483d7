# ncu --set full of one cfg4 k_condense_tc launch (line + opcode breakdown)
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_condense_tc -s 1 -c 1 -o gpurun_out/cond4_v9 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cond4_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/cond4_ncu.log
