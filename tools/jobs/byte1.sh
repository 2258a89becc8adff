SVB200_BYTE_PHASE_SKIP=1 timeout 900 python -m pytest tests/test_gpu_byte.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider > gpurun_out/byte_tests.log 2>&1; echo "rc=$?" >> gpurun_out/byte_tests.log; tail -2 gpurun_out/byte_tests.log
for sk in 0 1; do SVB200_BYTE_PHASE_SKIP=$sk timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -2; done
SVB200_BYTE_PHASE_SKIP=1 BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -12
timeout 600 python tools/byte_probe.py 32 adder 2>&1 | tail -2
timeout 300 python - <<'PY'
import subprocess, sys, json
sys.path.insert(0, ".")
import bench
print(bench.cold_e2e(33, 9, 0, 12))
PY
