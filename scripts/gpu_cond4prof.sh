#!/bin/bash
# K-COND at cfg4: launch geometry + one ncu --set full capture with source lines
GM_TC_DEBUG=1 timeout 300 python bench.py --workload cfg4 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -m2 "k_condense:"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_condense_tc -c 1 -o gpurun_out/full_cond_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
