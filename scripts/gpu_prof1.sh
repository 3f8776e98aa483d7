python scripts/profile_stages.py --M 1000 --N 20 --reps 6 > gpurun_out/prof_cfg3.log 2>&1; echo rc=$?
python scripts/profile_stages.py --M 10 --N 10 --reps 4 >> gpurun_out/prof_cfg3.log 2>&1
cat gpurun_out/prof_cfg3.log
python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/ncu_cfg3.log 2>&1; echo ncu rc=$?
