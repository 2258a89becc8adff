timeout 1500 python -m pytest tests/test_gpu_byte.py tests/test_gpu_ladder.py tests/test_gpu_fp.py -q -x -p no:cacheprovider > gpurun_out/bkc2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bkc2_tests.log
SVB200_TIME_BYTE_PASSES=1 BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 bench > gpurun_out/bkc2_bench.log 2>&1; grep -E "H\((7|6|5|4|3|2|1|0),\)" gpurun_out/bkc2_bench.log | head -8; tail -2 gpurun_out/bkc2_bench.log
BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 adder > gpurun_out/bkc2_adder.log 2>&1; tail -2 gpurun_out/bkc2_adder.log
