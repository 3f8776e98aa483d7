GM_LIB_PATH=$PWD/paper_2602_17601_b200/lib/ab/b.so timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_reference_dropin.py -q -p no:cacheprovider > gpurun_out/pytest_abqp.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/pytest_abqp.log | head -8
bash scripts/ab_cfg3.sh 3
