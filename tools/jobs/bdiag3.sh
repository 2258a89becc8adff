timeout 1500 python -m pytest tests/test_gpu_byte.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider > gpurun_out/bdiag3_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bdiag3_tests.log
BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 adder > gpurun_out/bdiag3_adder.log 2>&1; sed -n 20,24p gpurun_out/bdiag3_adder.log; tail -2 gpurun_out/bdiag3_adder.log
timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -1
