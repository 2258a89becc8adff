timeout 900 python -m pytest tests/test_gpu_byte.py tests/test_fp32_round.py -q -x -p no:cacheprovider > gpurun_out/byte3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/byte3_tests.log; tail -2 gpurun_out/byte3_tests.log
timeout 600 python tools/byte_probe.py 32 bench 2>&1 | tail -2
timeout 600 python tools/byte_probe.py 32 adder 2>&1 | tail -2
for r in 3 4; do SVB200_F32_ROUND=$r SVB200_JIT=1 timeout 900 python -m pytest tests/test_gpu_jit.py -q -x -p no:cacheprovider -k fp32 2>&1 | tail -1; done
for r in 3 4; do SVB200_F32_ROUND=$r timeout 900 python bench.py --steps 10 --warmup 3 --tier-n 0 --no-cpu --e2e-steps 0 --adder 0 --byte-n 0 --parity 0 --single-gate 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('round', $r, d['ms_per_step'], d['fp32']['ms_per_step'], d['fp32']['pass_GBps'], d['roofline']['fp64_aware'])"; done
