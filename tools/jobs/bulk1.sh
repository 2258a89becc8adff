# bulk tile loads: parity first (JIT passes, engine, ladder), then per-pass timing A/B
SVB200_JIT=1 timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_fp.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/bulk1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/bulk1_tests.log
SVB200_BULK=0 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_bulk0.jsonl 2>&1; tail -1 gpurun_out/pm_bulk0.jsonl
SVB200_BULK=1 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_bulk1.jsonl 2>&1; tail -1 gpurun_out/pm_bulk1.jsonl
for b in 0 1; do SVB200_BULK=$b timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --tier-n 0 --adder 1 --byte-n 0 --parity 0 --single-gate 0 --fp32 0 --cold-e2e 0 > gpurun_out/bulk_bench$b.json 2>gpurun_out/bulk_bench$b.err; python -c "
import json; d=json.loads(open('gpurun_out/bulk_bench$b.json').read().strip().splitlines()[-1]); print('bulk $b', d['ms_per_step'], d['roofline']['frac'], d['roofline']['fp64_aware'], d['e2e']['value'], d['adder']['seconds'], d['clocks'])"; done
