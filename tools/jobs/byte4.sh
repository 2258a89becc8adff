timeout 900 python -m pytest tests/test_gpu_byte.py -q -x -p no:cacheprovider > gpurun_out/byte4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/byte4_tests.log; tail -2 gpurun_out/byte4_tests.log
timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -2
timeout 600 python tools/byte_probe.py 32 adder 2>&1 | tail -2
