timeout 300 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_condense_tmap -c 1 -o gpurun_out/full_tmap_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo "ncu rc=$?"
