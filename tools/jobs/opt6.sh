timeout 1500 python -m pytest tests/test_gpu_byte.py tests/test_gpu_ladder.py tests/test_gpu_jit.py tests/test_gpu_tier.py -q -p no:cacheprovider > gpurun_out/opt6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/opt6_tests.log; tail -3 gpurun_out/opt6_tests.log
timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -2
timeout 600 python tools/byte_probe.py 32 adder 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fp.py -q -p no:cacheprovider -k "torchrun and 2" 2>&1 | tail -2
