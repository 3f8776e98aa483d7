#!/bin/bash
# tcgen05 psi VJP (k_jac_psi_tc, linearize mode 0/2) vs the SIMT chain
# (k_jac_psi, mode 4): GPU tests, per-launch ncu times, short benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for w in cfg3 cfg5 cfg4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_jac_psi -c 1 \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'k_jac_psi|duration' | tail -2 | sed "s/^/tc $w /"
  GM_LINEARIZE_MODE=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_jac_psi -c 1 \
    python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'k_jac_psi|duration' | tail -2 | sed "s/^/simt $w /"
done
for w in cfg3 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/jp_$w.json
  python -c "import json;d=json.load(open('gpurun_out/jp_$w.json'));print('$w', d['ms_per_step'], d.get('stage_ms'))"
done
