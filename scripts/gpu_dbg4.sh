for c in "1000 20 3 chain:256,4,2" "1000 20 3 chain:512,4,2" "1000 20 1 chain:256,4,2"; do
  args=${c%%:*}; cfg=${c##*:}
  r=$(GM_TC_DEBUG=1 GM_TC_CFG=$cfg timeout 120 python scripts/dbg_fused_case.py $args 2>&1 | grep -E "^ok|Error|assert|k_condense:" | sort -u | head -3 | cut -c1-120)
  echo "$args $cfg -> $r"
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
GM_TC_DEBUG=1 timeout 300 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "k_condense:" | sort -u | head -2
