timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python scripts/profile_stages.py --M 1000 --N 20 --reps 5 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prof.csv python scripts/profile_stages.py --M 1000 --N 20 --reps 3 > gpurun_out/launch_prof.log 2>&1; echo rc=$?
python scripts/summarize_launches.py gpurun_out/launches_prof.csv
