for c in "1600 20 1 chain:256,4,1" "1600 20 1 chain:256,4,2" "2000 20 1 chain:256,4,1" "1000 20 3 chain:256,4,2" "1000 20 3 chain:512,4,2"; do
  args=${c%%:*}; cfg=${c##*:}
  r=$(GM_TC_CFG=$cfg timeout 120 python scripts/dbg_fused_case.py $args 2>&1 | grep -E "^ok|Error|assert" | head -1 | cut -c1-80)
  echo "$args $cfg -> $r"
done
