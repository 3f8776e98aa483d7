for c in "1000 20 2 chain" "1000 20 3 chain" "1000 5 3 chain" "400 20 3 chain" "2000 20 3 chain" "1000 20 4 chain" "1000 20 6 chain" "391 12 3 mesh"; do
  r=$(GM_TC_CFG=256,4,2 timeout 120 python scripts/dbg_fused_case.py $c 2>&1 | grep -E "^ok|Error|assert" | head -1 | cut -c1-80)
  echo "$c -> $r"
done
