timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_stages.py -x -q 2>&1 | tail -3
timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 4 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python scripts/profile_stages.py --M 1000 --N 20 --reps 3 > gpurun_out/launch_prof.log 2>&1; echo rc=$?
python scripts/summarize_launches.py gpurun_out/launches_prof.csv | head -5
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_condense_fused -s 1 -c 1 -o gpurun_out/fused_prof python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/fused_ncu.log 2>&1; echo ncu rc=$?
