timeout 1200 python -m pytest tests/test_gpu_fp.py -q -x -p no:cacheprovider -k "combined or adder or kernels_match" > gpurun_out/comb1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/comb1_tests.log
timeout 900 python tools/adder_combine_probe.py 16
