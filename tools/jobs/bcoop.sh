timeout 1200 python -m pytest tests/test_gpu_byte.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider > gpurun_out/bcoop_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bcoop_tests.log
SVB200_TIME_BYTE_PASSES=1 BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 bench > gpurun_out/bcoop_bench.log 2>&1; tail -40 gpurun_out/bcoop_bench.log
BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 adder > gpurun_out/bcoop_adder.log 2>&1; tail -3 gpurun_out/bcoop_adder.log
