timeout 600 python -m pytest tests/test_experiments.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python -m paper_2602_17601_b200.experiments scaling --out gpurun_out/scaling > gpurun_out/scaling.log 2>&1; echo "scaling rc=$?"; cat gpurun_out/scaling/scaling.csv gpurun_out/scaling/scaling_device.csv
