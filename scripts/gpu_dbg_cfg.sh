T='tests/test_gpu_fused.py::test_fused_matches_two_kernel_path[0-chain1000-20-6-6-3]'
for env in "GM_TC_CFG=512,8,1" "GM_TC_CFG=256,4,2" "GM_TC_CFG=256,4,2 GM_TC_PREFETCH=0" "GM_TC_CFG=256,8,1" "GM_TC_CFG=256,4,1" "GM_TC_CFG=512,4,1" "GM_TC_CFG=256,8,2"; do
  r=$(env $env timeout 120 python -m pytest "$T" -x -q -p no:cacheprovider 2>&1 | grep -E "passed|failed" | tail -1)
  echo "$env -> $r"
done
