timeout 1800 python -m pytest tests/test_gpu_fp.py tests/test_gpu_ladder.py tests/test_gpu_jit.py tests/test_gpu_tier.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/sup1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sup1_tests.log
timeout 900 python tools/adder_combine_probe.py 16
SVB200_SUPPORT=0 timeout 900 python tools/adder_combine_probe.py 16
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --tier-n 0 --adder 0 --byte-n 0 --parity 0 --single-gate 0 --fp32 0 --cold-e2e 0 > gpurun_out/sup1_bench.json 2>gpurun_out/sup1_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/sup1_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['e2e'])[:600])"
