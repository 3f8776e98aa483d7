timeout 120 python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/plain_lin.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_linearize -s 1 -c 1 -o gpurun_out/lin_prof python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/lin_ncu.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cost_partial -s 1 -c 1 -o gpurun_out/hg_prof python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/hg_ncu.log 2>&1; echo ncu2 rc=$?
