timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python scripts/profile_stages.py --M 1000 --N 20 --reps 3 > gpurun_out/launch_prof.log 2>&1; echo rc=$?
python scripts/summarize_launches.py gpurun_out/launches_prof.csv
