timeout 600 python -m pytest tests/test_gpu_tier.py tests/test_tier.py -q -x -p no:cacheprovider > gpurun_out/pytest_tier.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tier.log
tail -5 gpurun_out/pytest_tier.log
timeout 600 python tools/tier_bench.py 30 10 1 > gpurun_out/tier30.json 2>&1; tail -3 gpurun_out/tier30.json
timeout 900 python tools/tier_bench.py 34 168 4 > gpurun_out/tier34.json 2>&1; tail -3 gpurun_out/tier34.json
