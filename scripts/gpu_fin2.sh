#!/bin/bash
# K-RS epilogue variants: per-launch time of k_finish_states at cfg5 / cfg4 for
# each GM_FIN_MODE, then the GPU test suite on the default.
mkdir -p gpurun_out
for m in 0 1 2 3; do
  for w in cfg5 cfg4; do
    GM_FIN_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_finish_states -c 2 \
      python bench.py --workload $w --steps 1 --warmup 0 --no-cpu-baseline 2>&1 | grep -E 'duration|bytes_read' | tail -2 | sed "s/^/mode=$m $w /"
  done
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
