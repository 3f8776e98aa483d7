# K-QP cluster mode: QP tests, cfg3 bench with/without the helper CTA, phase profile
timeout 600 python -m pytest tests/test_gpu_stages.py -q -p no:cacheprovider -x -k "qp or chol or mpc_step or plugin" > gpurun_out/pytest_qpcl.log 2>&1; echo "pytest rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_qpcl.log | head -20
for cl in 1 0; do GM_QP_CLUSTER=$cl timeout 300 python bench.py --no-legs --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bench_qpcl_$cl.json 2> gpurun_out/bench_qpcl_$cl.err; echo "bench cl=$cl rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_qpcl_$cl.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['stage_ms'], d['config']['qp'])"; tail -2 gpurun_out/bench_qpcl_$cl.err; done
GM_QP_CLUSTER=1 timeout 300 python scripts/qp_phases.py cfg3 > gpurun_out/qp_phases_cl.txt 2>&1; head -14 gpurun_out/qp_phases_cl.txt
