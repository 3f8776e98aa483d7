for m in 1 2; do echo "lin mode $m"; GM_LINEARIZE_MODE=$m timeout 300 python scripts/profile_stages.py --M 10000 --N 20 --reps 4 2>&1 | tail -2; done
for m in 1 2; do echo "lin mode $m M=1000"; GM_LINEARIZE_MODE=$m timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 4 2>&1 | tail -2; done
