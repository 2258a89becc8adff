free -g
timeout 600 python -m pytest tests/test_gpu_tier.py tests/test_tier.py -q -x -p no:cacheprovider > gpurun_out/pytest_tier.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tier.log
tail -30 gpurun_out/pytest_tier.log
nvcc -O2 -o tools/pin_probe tools/pin_probe.cu -lpthread 2>/dev/null; timeout 300 tools/pin_probe 16 > gpurun_out/pin_probe.json 2>&1; cat gpurun_out/pin_probe.json
timeout 600 python tools/tier_bench.py 30 10 1 > gpurun_out/tier30.json 2>&1; cat gpurun_out/tier30.json | tail -5
