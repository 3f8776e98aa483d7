#!/bin/bash
# round-1 evidence pass v8 (DMMA forward chains): GPU tests, smoke, benches (cfg3 default + reference arm, cfg2, cfg4, cfg5), launch lists, ncu --set full of the forward chains and the top kernels, 1e3..1e4 sweep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-steps 4 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
for w in cfg2 cfg4 cfg5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-steps 2 2>/dev/null | tail -1 > gpurun_out/bench_$w.json; echo "bench $w: $(python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print(d['ms_per_step'], d['value'], d['unit'])")"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>/dev/null; head -14 gpurun_out/launches.txt
for w in cfg4 cfg5; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python scripts/summarize_launches.py gpurun_out/launches_$w.csv > gpurun_out/launches_$w.txt 2>/dev/null; done
for k in k_fwd_chain_mma k_solve_qp k_condense_tc; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/full8_$k python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > /dev/null 2>&1; echo "ncu $k rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fwd_chain_mma -c 2 -o gpurun_out/full8_fwd_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu fwd cfg5 rc=$?"
timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases.txt 2>&1
timeout 900 python -c "
import sys; sys.path.insert(0,'.')
from paper_2602_17601_b200 import experiments as ex
rows = ex.run_device_sweep([1000, 2000, 5000, 10000], reps=3)
print('node_count,linearize_ms,condense_ms,solve_ms,step_ms,status,iterations')
for d in rows: print(','.join(str(d[k]) for k in ['node_count','linearize_ms','condense_ms','solve_ms','step_ms','status','iterations']))
" > gpurun_out/sweep_big.csv 2> /dev/null; cat gpurun_out/sweep_big.csv
