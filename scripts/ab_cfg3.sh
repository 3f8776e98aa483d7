# A/B/... of library builds on the same box: every paper_2602_17601_b200/lib/ab/*.so
# usage: bash scripts/ab_cfg3.sh [rounds] [bench args]
R=${1:-3}; shift
ARGS=${@:---no-legs --no-cpu-baseline}
for i in $(seq $R); do for f in paper_2602_17601_b200/lib/ab/*.so; do
  v=$(basename $f .so)
  GM_LIB_PATH=$PWD/$f timeout 300 python bench.py $ARGS > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d.get('stage_ms', d.get('stage_ms_per_wave', {}));print('$v', round(d['ms_per_step'],4), {k: round(v,3) for k,v in s.items()})"
done; done
