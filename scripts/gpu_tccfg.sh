for c in "512,8,1" "256,4,2" "256,8,1" "384,8,1" "128,4,3" "256,2,3"; do
  r=$(GM_TC_CFG=$c timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_condense_tc -c 1 python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration' | head -1)
  r4=$(GM_TC_CFG=$c timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_condense_tc -c 1 python bench.py --workload cfg4 --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration' | head -1)
  r3=$(GM_TC_CFG=$c timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_condense_tc -c 1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration' | head -1)
  echo "$c | cfg5 $r | cfg4 $r4 | cfg3 $r3"
done
