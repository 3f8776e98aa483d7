GM_LIB_PATH=$PWD/paper_2602_17601_b200/lib/ab/b.so timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "lin or stage or mesh" > gpurun_out/pytest_ablin.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ablin.log
bash scripts/ab_cfg3.sh 2 --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline
bash scripts/ab_cfg3.sh 2 --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline
