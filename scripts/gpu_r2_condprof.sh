# K-COND (SIMT fused, the round-2 default) at cfg4 and cfg5: one ncu --set full capture each
timeout 300 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_condense_tma -c 1 -o gpurun_out/full_tma3_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
timeout 300 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_condense_tma -c 1 -o gpurun_out/full_tma3_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo "ncu5 rc=$?"
ls -la gpurun_out/*.ncu-rep
