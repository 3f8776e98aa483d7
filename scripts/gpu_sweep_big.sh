timeout 900 python -c "
import sys; sys.path.insert(0,'.')
from paper_2602_17601_b200 import experiments as ex
rows = ex.run_device_sweep([1000, 2000, 5000, 10000], reps=3)
print('node_count,linearize_ms,condense_ms,solve_ms,step_ms,status,iterations')
for d in rows: print(','.join(str(d[k]) for k in ['node_count','linearize_ms','condense_ms','solve_ms','step_ms','status','iterations']))
" > gpurun_out/sweep_big.csv 2> gpurun_out/sweep_big.err; echo rc=$?; cat gpurun_out/sweep_big.csv; tail -3 gpurun_out/sweep_big.err
