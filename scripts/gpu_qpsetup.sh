#!/bin/bash
# K-QP setup rewritten as flat passes + warp compactions: GPU tests, phase
# breakdown, cfg3 / cfg4 benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python scripts/qp_phases.py 2>&1 | tail -20
for w in cfg3 cfg4; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/qs_$w.json
  python -c "import json;d=json.load(open('gpurun_out/qs_$w.json'));print('$w', d['ms_per_step'], d['value'], d.get('stage_ms'))"
done
