# WavePipeline: GPU tests + cfg4 bench (e2e through the pipeline)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 --cpu-steps 2 2>gpurun_out/bench_cfg4.err | tail -1 > gpurun_out/bench_cfg4.json; echo "bench cfg4: $(python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print(d['ms_per_step'], d['value'], d['e2e'])")"; tail -3 gpurun_out/bench_cfg4.err
