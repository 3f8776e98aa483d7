#!/bin/bash
# fp64 forward chains on DMMA (k_fwd_chain_mma, linearize mode 0/2) vs the
# per-row SIMT chains (k_fwd_chain, mode 4): GPU tests, per-launch ncu, benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for w in cfg3 cfg5 cfg4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fwd_chain -c 2 \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration' | tail -2 | sed "s/^/mma $w /"
  GM_LINEARIZE_MODE=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fwd_chain -c 2 \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration' | tail -2 | sed "s/^/simt $w /"
done
for w in cfg3 cfg5 cfg4; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fm_$w.json
  python -c "import json;d=json.load(open('gpurun_out/fm_$w.json'));print('$w', d['ms_per_step'], d['value'], d.get('stage_ms'))"
done
