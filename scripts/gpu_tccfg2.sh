#!/bin/bash
# K-COND launch-config sweep (GM_TC_CFG=threads,sc,cps) at cfg4 / cfg5 / cfg3
for cfg in 512,8,1 256,8,2 256,4,2 128,4,4 512,4,1 512,12,1 256,6,2; do
  for w in cfg4 cfg5 cfg3; do
    GM_TC_DEBUG=1 GM_TC_CFG=$cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_condense_tc -c 1 \
      python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/tc_$w.log 2>&1
    echo "$cfg $w $(grep -m1 -o 'occ=[0-9]* smem=[0-9]*' gpurun_out/tc_$w.log) $(grep -E 'gpu__time_duration' gpurun_out/tc_$w.log | tail -1 | awk '{print $(NF-1), $NF}')"
  done
done
rm -f gpurun_out/tc_*.log
