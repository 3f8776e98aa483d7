# round-1 evidence pass v5: GPU tests, smoke, benches (cfg3 default + reference arm, cfg2, cfg4, cfg5), launch lists, ncu --set full of the top kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-steps 4 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"
for w in cfg2 cfg4 cfg5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-steps 2 2>/dev/null | tail -1 > gpurun_out/bench_$w.json; echo "bench $w: $(cut -c1-400 gpurun_out/bench_$w.json)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>/dev/null; head -8 gpurun_out/launches.txt
for w in cfg4 cfg5; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python scripts/summarize_launches.py gpurun_out/launches_$w.csv > gpurun_out/launches_$w.txt 2>/dev/null; done
for k in k_solve_qp k_linearize k_condense_tc; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_$k python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > /dev/null 2>&1; echo "ncu $k rc=$?"
done
for k in k_condense_tc k_jac_psi k_fwd_chain; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full_cfg5_$k python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg5 $k rc=$?"
done
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1
