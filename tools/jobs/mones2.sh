SVB200_MEASURE_ONES_PASS=1 timeout 1200 python -m pytest tests/test_gpu_fp.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/mones2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mones2_tests.log
for o in 0 1 0 1; do SVB200_MEASURE_ONES_PASS=$o timeout 600 python tools/measure_probe.py 33; done
