for i in 1 2 3; do timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]);print('cfg3', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])"; done
nvidia-smi --query-gpu=name,pci.bus_id,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
