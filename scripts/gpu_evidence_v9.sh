#!/bin/bash
# round-1 final evidence pass v9: GPU tests, smoke, benches (cfg3 default + reference arm, cfg2, cfg4, cfg5), default-bench launch list, ncu --set full of k_condense_tc (cfg3)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-steps 4 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
for w in cfg2 cfg4 cfg5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-steps 2 2>/dev/null | tail -1 > gpurun_out/bench_$w.json; echo "bench $w: $(python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print(d['ms_per_step'], d['value'], d['unit'])")"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>/dev/null; head -14 gpurun_out/launches.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_condense_tc -s 1 -c 1 -o gpurun_out/full9_k_condense_tc python scripts/profile_stages.py --M 1000 --N 20 --reps 2 > /dev/null 2>&1; echo "ncu cond rc=$?"
