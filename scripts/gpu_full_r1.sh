# round-1 evidence pass: GPU tests, K-QP phase profile, bench, launch list, ncu --set full of the 3 top kernels
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1; head -14 gpurun_out/qp_phases.txt
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-steps 4 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python scripts/summarize_launches.py gpurun_out/launches.csv | head -14
for k in k_solve_qp k_linearize k_condense_fused; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$k python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
