timeout 120 python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/plain_fused.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_condense_fused -s 1 -c 1 -o gpurun_out/fused_prof python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/fused_ncu.log 2>&1; echo ncu rc=$?
