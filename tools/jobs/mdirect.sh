timeout 1200 python -m pytest tests/test_gpu_fp.py tests/test_gpu_ladder.py tests/test_gpu_tier.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/mdirect_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mdirect_tests.log
for d in 0 1; do SVB200_MEASURE_DIRECT=$d timeout 600 python tools/measure_probe.py 33; done
for d in 0 1; do SVB200_MEASURE_DIRECT=$d timeout 600 python tools/e2e_probe.py 33 | tail -1; done
