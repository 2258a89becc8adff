timeout 1200 python -m pytest tests/test_gpu_fp.py tests/test_gpu_jit.py -q -x -p no:cacheprovider -k "combined or adder or bit_exact" > gpurun_out/comb2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/comb2_tests.log
timeout 900 python tools/adder_combine_probe.py 16
